"""Copy the judged evidence from gpurun_out/evidence/ into profiles/ (round tag
argv[1], default r01): bench lines, launch lists, ncu --set full summaries,
per-kernel DRAM traffic for bench.py's roofline.traffic."""
import json
import os
import shutil
import subprocess
import sys

tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
src = "gpurun_out/evidence"
dst = "profiles"
for f in ["bench.json", "bench_cfg5.json", "bench_cfg4.json", "bench_cfg1.json", "gpu.txt",
          "launches.csv", "launches_cfg5.csv"]:
    if os.path.exists(os.path.join(src, f)):
        shutil.copy(os.path.join(src, f), os.path.join(dst, f"{tag}_{f}"))
summ = {}
for rep, name in [("k1_full", "k1_cfg2_fwd_ws"), ("k1_cfg5_full", "k1_cfg5_rsw_mlp_tc"),
                  ("k2_full", "k2_train")]:
    path = os.path.join(src, rep + ".ncu-rep")
    if not os.path.exists(path):
        continue
    out = subprocess.run([sys.executable, "tools/ncu_summary.py", path], capture_output=True,
                         text=True).stdout
    with open(os.path.join(dst, f"{tag}_{name}_ncu.json"), "w") as fh:
        fh.write(out)
    lines = subprocess.run([sys.executable, "tools/ncu_lines.py", path, "30"], capture_output=True,
                           text=True).stdout
    with open(os.path.join(dst, f"{tag}_{name}_ncu_lines.txt"), "w") as fh:
        fh.write(lines)
    summ[name] = json.loads(out)
# bench.py roofline.traffic: DRAM bytes per launch of the dominant kernel
traffic = {"_note": "dram__bytes_read.sum + dram__bytes_write.sum per launch of the dominant "
                    "kernel (ncu --set full, profiles/*_ncu.json)"}
if "k1_cfg2_fwd_ws" in summ:
    traffic["cfg2_deepffm_fwd"] = summ["k1_cfg2_fwd_ws"][0]["dram_bytes_per_launch"]
if "k1_cfg5_rsw_mlp_tc" in summ:
    ks = summ["k1_cfg5_rsw_mlp_tc"]
    traffic["cfg5_large_bf16_per_slice"] = sum(k["dram_bytes_per_launch"] for k in ks)
    traffic["cfg5_large_bf16"] = ks[0]["dram_bytes_per_launch"]  # the gather (dominant) kernel
with open(os.path.join(dst, "ncu_traffic.json"), "w") as fh:
    json.dump(traffic, fh, indent=1)
print("copied; traffic:", traffic)
