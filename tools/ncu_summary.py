"""Summarise an ncu --set full report into the numbers profiles/ records."""
import csv
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "launch__shared_mem_per_block_dynamic"]


def summarise(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u = rows[0], rows[1]
    res = []
    for v in rows[2:]:
        d = dict(zip(h, v))
        ent = {"kernel": d.get("Kernel Name", "")[:120]}
        for k in KEYS:
            if k in d:
                ent[k] = f"{d[k]} {u[h.index(k)]}".strip()
        st = [(float(d[k].replace(",", "") or 0), k) for k in h
              if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued")]
        tot = sum(s for s, _ in st) or 1.0
        ent["stall_top"] = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): round(100 * s / tot, 1)
                            for s, k in sorted(st, reverse=True)[:6]}
        rb = float(d.get("dram__bytes_read.sum", "0").replace(",", "") or 0)
        wb = float(d.get("dram__bytes_write.sum", "0").replace(",", "") or 0)
        unit_r = u[h.index("dram__bytes_read.sum")]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit_r, 1)
        scale_w = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(
            u[h.index("dram__bytes_write.sum")], 1)
        ent["dram_bytes_per_launch"] = rb * scale + wb * scale_w
        res.append(ent)
    return res


if __name__ == "__main__":
    print(json.dumps(summarise(sys.argv[1]), indent=1))
