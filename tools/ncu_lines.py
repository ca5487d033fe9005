"""Per-source-line warp-stall samples / instructions from an ncu report
(`--page source --print-source cuda,sass`): top lines by stall samples."""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                      "cuda,sass"], capture_output=True, text=True).stdout
fname, acc, tot_s, tot_i = "?", [], 0, 0
for r in csv.reader(out.splitlines()):
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) < 8 or r[0] == "Line No" or r[2] != "-":
        continue
    try:
        s, i = int(r[4]), int(r[7])
    except ValueError:
        continue
    tot_s += s
    tot_i += i
    acc.append((s, i, f"{fname}:{r[0]}", r[1].strip()[:90]))
acc.sort(reverse=True)
print(f"total samples {tot_s}, warp-instructions {tot_i}")
for s, i, loc, src in acc[:top]:
    print(f"{100*s/max(tot_s,1):5.1f}% smp {100*i/max(tot_i,1):5.1f}% inst  {loc:22s} {src}")
