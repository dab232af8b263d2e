"""Summarise an ncu --page source --print-source cuda,sass CSV by source line:
warp-stall samples per line (top N). Usage: ncu_lines.py rep.ncu-rep [N]"""
import csv, subprocess, sys
rep = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
path = None
items = []
tot = 0
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        path = r[1].split("/")[-1]
        continue
    if len(r) < 6 or r[0] in ("Line No", "Function Name"):
        continue
    if r[2] != "-":  # sass rows
        continue
    try:
        w = int(r[4])
    except ValueError:
        continue
    tot += w
    items.append((w, f"{path}:{r[0]}", r[1][:100]))
items.sort(reverse=True)
print("total samples", tot)
for w, loc, s in items[:N]:
    print(f"{w:7d} {100 * w / max(tot, 1):5.1f}% {loc:24s} {s}")
