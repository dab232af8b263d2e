"""Summarise an ncu capture by CUDA source line: warp-stall samples and executed
(warp) instructions per line, top N by instructions and by stalls.
Usage: ncu_lines.py rep.ncu-rep [N]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
path, hdr = None, None
items = []
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        path = r[1].split("/")[-1]
        continue
    if len(r) >= 2 and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 9 or r[0] in ("", "Function Name"):
        continue
    try:
        stall = int(r[hdr.index("Warp Stall Sampling (All Samples)")])
        inst = int(r[hdr.index("Instructions Executed")])
        tinst = int(r[hdr.index("Thread Instructions Executed")])
    except (ValueError, IndexError):
        continue
    items.append((inst, stall, tinst, f"{path}:{r[0]}", r[1][:90]))
ti = sum(x[0] for x in items) or 1
ts = sum(x[1] for x in items) or 1
tt = sum(x[2] for x in items)
print(f"total warp instructions {ti}, thread instructions {tt} (SIMT {tt / (32 * ti):.2f}), stall samples {ts}")
print("--- by instructions")
for inst, stall, tinst, loc, s in sorted(items, reverse=True)[:N]:
    print(f"{inst:11d} {100 * inst / ti:5.1f}%  simt {tinst / max(32 * inst, 1):.2f}  stall {100 * stall / ts:5.1f}%  {loc:26s} {s}")
print("--- by stalls")
for inst, stall, tinst, loc, s in sorted(items, key=lambda x: -x[1])[:N]:
    print(f"{inst:11d} {100 * inst / ti:5.1f}%  simt {tinst / max(32 * inst, 1):.2f}  stall {100 * stall / ts:5.1f}%  {loc:26s} {s}")
