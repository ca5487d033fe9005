"""Run ON the GPU box after tools/evidence_r2.sh: summarise every ncu report of
gpurun_out/evidence/ into small text/json files (tools/ncu_summary.py,
tools/ncu_lines.py), build the roofline-traffic record (DRAM bytes per launch of
the dominant kernel, tied to the libdffm.so sha) from the launch lists, and
delete the reports not listed in KEEP (so the copy-back stays small)."""
import csv
import glob
import hashlib
import json
import os
import subprocess
import sys
from collections import defaultdict

src = "gpurun_out/evidence"
keep = set(os.environ.get("KEEP", "").split())
for rep in sorted(glob.glob(os.path.join(src, "*.ncu-rep"))):
    base = rep[:-len(".ncu-rep")]
    out = subprocess.run([sys.executable, "tools/ncu_summary.py", rep], capture_output=True,
                         text=True).stdout
    open(base + "_ncu.json", "w").write(out)
    lines = subprocess.run([sys.executable, "tools/ncu_lines.py", rep, "40"], capture_output=True,
                           text=True).stdout
    open(base + "_ncu_lines.txt", "w").write(lines)
    if os.path.basename(base) not in keep:
        os.remove(rep)


def per_launch(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    if not rows:
        return {}
    h = rows[0]
    ii, ki, mi, vi = (h.index(c) for c in ("ID", "Kernel Name", "Metric Name", "Metric Value"))
    per = defaultdict(dict)
    for r in rows[1:]:
        per[int(r[ii])][r[mi]] = float(r[vi].replace(",", ""))
        per[int(r[ii])]["k"] = r[ki].split("(")[0].split("<")[0].replace("void ", "")
    by = defaultdict(lambda: [0, 0.0, 0.0])
    for d in per.values():
        b = d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
        by[d["k"]][0] += 1
        by[d["k"]][1] += d.get("gpu__time_duration.sum", 0) / 1e6
        by[d["k"]][2] += b
    return {k: {"launches": v[0], "ms": round(v[1], 4), "dram_bytes": v[2]} for k, v in by.items()}


sys.path.insert(0, os.getcwd())
from paper_2407_10115_b200 import _lib  # noqa: E402
bid = _lib.lib().dffm_build_id().decode()
traffic = {"_note": "roofline.traffic of bench.py: dram__bytes_read.sum + dram__bytes_write.sum "
                    "per launch of the dominant kernel (fwd_rsw_kernel, the K1 v8 row-ring "
                    "gather), averaged over the launches of ONE forward step (ncu launch list "
                    "of tools/one_forward.py, NVTX range 'step', --clock-control none; "
                    "cold-cache serialised replay); valid only for the libdffm.so whose build id "
                    "(dffm_build_id: digest of its sources) is recorded", "captures": {}}
for w, key in [("cfg2", "cfg2_deepffm_fwd"), ("cfg5", "cfg5_large_bf16")]:
    path = os.path.join(src, f"launches_{w}.csv")
    if not os.path.exists(path):
        continue
    by = per_launch(path)
    g = by.get("dffm::fwd_rsw_kernel")
    if g:
        traffic["captures"][key] = {"build_id": bid, "dram_bytes_per_launch": g["dram_bytes"] / g["launches"],
                                    "launches": g["launches"], "source": f"profiles/r02_launches_{w}.csv",
                                    "step_kernels": by}
json.dump(traffic, open(os.path.join(src, "ncu_traffic.json"), "w"), indent=1)
print(json.dumps(traffic)[:800])
