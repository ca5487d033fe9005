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
for f in ["bench.json", "bench_cfg5.json", "bench_cfg4.json", "bench_cfg1.json",
          "bench_parse.json", "gpu.txt", "launches_cfg2.csv", "launches_cfg5.csv"]:
    if os.path.exists(os.path.join(src, f)):
        shutil.copy(os.path.join(src, f), os.path.join(dst, f"{tag}_{f}"))
summ = {}
for rep, name in [("k1_cfg2_full", "k1_cfg2_rsw_mlp_tc"), ("k1_cfg5_full", "k1_cfg5_rsw_mlp_tc"),
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
# bench.py roofline.traffic: DRAM bytes of ONE forward step (every launch inside the
# NVTX "step" range of tools/one_forward.py), from the launch lists
import csv
from collections import defaultdict


def step_traffic(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    if not rows:
        return None, {}
    h = rows[0]
    ii, ki, mi, vi = (h.index(c) for c in ("ID", "Kernel Name", "Metric Name", "Metric Value"))
    per = defaultdict(dict)
    for r in rows[1:]:
        per[int(r[ii])][r[mi]] = float(r[vi].replace(",", ""))
        per[int(r[ii])]["k"] = r[ki].split("(")[0].split("<")[0].replace("void ", "")
    tot, by = 0.0, defaultdict(lambda: [0, 0.0, 0.0])
    for d in per.values():
        b = d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
        tot += b
        by[d["k"]][0] += 1
        by[d["k"]][1] += d.get("gpu__time_duration.sum", 0) / 1e6
        by[d["k"]][2] += b
    return tot, {k: {"launches": v[0], "ms": round(v[1], 4), "dram_bytes": v[2]} for k, v in by.items()}


traffic = {"_note": "dram__bytes_read.sum + dram__bytes_write.sum summed over every kernel "
                    "of one forward step (ncu launch list of tools/one_forward.py, NVTX range "
                    "'step'; cold-cache serialised replay)"}
for w, key in [("cfg2", "cfg2_deepffm_fwd"), ("cfg5", "cfg5_large_bf16")]:
    path = os.path.join(src, f"launches_{w}.csv")
    if os.path.exists(path):
        tot, by = step_traffic(path)
        traffic[key] = tot
        traffic[key + "_kernels"] = by
with open(os.path.join(dst, "ncu_traffic.json"), "w") as fh:
    json.dump(traffic, fh, indent=1)
print("copied; traffic:", json.dumps(traffic)[:600])
