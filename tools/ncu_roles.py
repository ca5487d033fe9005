"""Role-level view of an ncu report of a warp-specialised kernel (SASS page): groups
instructions by how often each executes (a role's per-item code executes once per item
per warp of the role), and lists every barrier / wait instruction with its samples."""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
hdr = [i for i, r in enumerate(rows) if r and r[0] == "Address"][0]
h = rows[hdr]
isrc, ismp, iex = h.index("Source"), h.index("# Samples"), h.index("Instructions Executed")
data = [(r[isrc], int(r[ismp]), int(r[iex])) for r in rows[hdr + 1:] if len(r) > iex]
print("instructions", len(data), "samples", sum(d[1] for d in data), "executed", sum(d[2] for d in data))
unit = float(sys.argv[2]) if len(sys.argv) > 2 else 1e6
cl, sm, n = Counter(), Counter(), Counter()
for s, smp, ex in data:
    key = round(ex / unit, 2)
    cl[key] += ex; sm[key] += smp; n[key] += 1
for k in sorted(cl, key=lambda k: -cl[k])[:16]:
    print(f"exec/instr {k:8.2f}  n_instr {n[k]:4d} total_exec {cl[k]/1e6:8.1f}M samples {sm[k]}")
for i, (s, smp, ex) in enumerate(data):
    if any(t in s for t in ("SYNCS", "BAR.", "UBLKCP", "DEPBAR")) and ex > 1000:
        print(i, s.strip()[:64], "smp", smp, "win4", sum(d[1] for d in data[i:i + 4]), "exec", ex)
