"""Copy the round-2 evidence (tools/evidence_r2.sh parts bench / launch / ncu, the cfg3
stream line and the final test / smoke logs) from gpurun_out/ into profiles/r02_*."""
import os
import shutil

src, fin, dst = "gpurun_out/evidence", "gpurun_out/final", "profiles"
plain = ["bench.json", "bench_cfg4.json", "bench_cfg1.json", "bench_parse.json", "bench_cfg3.json",
         "gpu.txt", "so_sha.txt", "launches_cfg5.csv", "launches_cfg2.csv", "launches_bench.csv"]
for f in plain:
    if os.path.exists(os.path.join(src, f)):
        shutil.copy(os.path.join(src, f), os.path.join(dst, "r02_" + f))
for rep, name in [("k1_cfg5_full", "k1_cfg5_rsw_mlp_tc"), ("k1_cfg2_full", "k1_cfg2_rsw_mlp_tc"),
                  ("k3_cfg4_full", "k3_cfg4_ctx_ring_mlp_tc"), ("k2_full", "k2_train")]:
    for suf in ("_ncu.json", "_ncu_lines.txt"):
        p = os.path.join(src, rep + suf)
        if os.path.exists(p):
            shutil.copy(p, os.path.join(dst, f"r02_{name}{suf}"))
if os.path.exists(os.path.join(src, "ncu_traffic.json")):
    shutil.copy(os.path.join(src, "ncu_traffic.json"), os.path.join(dst, "ncu_traffic.json"))
if os.path.exists("gpurun_out/cfg3_auc_series.json"):
    shutil.copy("gpurun_out/cfg3_auc_series.json", os.path.join(dst, "r02_cfg3_auc_series.json"))
for f, t in [("gpu_tests.txt", "r02_final_gpu_tests.txt"), ("smoke.txt", "r02_final_smoke.txt")]:
    if os.path.exists(os.path.join(fin, f)):
        shutil.copy(os.path.join(fin, f), os.path.join(dst, t))
print(sorted(x for x in os.listdir(dst) if x.startswith("r02_")))
