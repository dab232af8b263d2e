"""Condense ncu captures into the tracked summaries under profiles/.

    python scripts/ncu_summary.py <tag> gpurun_out/prof_<kernel>.ncu-rep ... [--launches gpurun_out/launches.csv]

Writes profiles/<tag>_<kernel>.txt (speed-of-light, memory, occupancy, FP64 pipe,
top source lines by warp-stall samples), profiles/<kernel>_ncu.json (dram bytes
per launch, read by bench.py as roofline.traffic) and, with --launches, the
per-kernel launch list summary profiles/<tag>_launches.txt.
"""
import csv
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sectors.sum",
        "lts__t_sectors_lookup_hit.sum", "lts__t_sectors_lookup_miss.sum", "l1tex__t_sectors.sum",
        "l1tex__t_sector_hit_rate.pct", "l1tex__texin_requests.sum", "smsp__inst_executed_op_texture.sum",
        "l1tex__t_bytes.sum", "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__instruction_throughput.avg.pct_of_peak_sustained_active",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed"]


def ncu(*args):
    return subprocess.run(["ncu", *args], capture_output=True, text=True).stdout


def raw(rep):
    rows = list(csv.reader(ncu("-i", rep, "--page", "raw", "--csv").splitlines()))
    h, u = rows[0], rows[1]
    out = []
    for v in rows[2:]:
        d = {}
        for i, n in enumerate(h):
            if n in KEYS or n == "Kernel Name":
                d[n] = (v[i], u[i])
        out.append(d)
    return out


def lines(rep, n=30):
    rows = list(csv.reader(ncu("-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass").splitlines()))
    path, items, tot = None, [], 0
    for r in rows:
        if len(r) >= 2 and r[0] == "File Path":
            path = r[1].split("/")[-1]
            continue
        if len(r) < 6 or r[0] in ("Line No", "Function Name") or r[2] != "-":
            continue
        try:
            w = int(r[4])
        except ValueError:
            continue
        tot += w
        items.append((w, f"{path}:{r[0]}", r[1].strip()[:100]))
    items.sort(reverse=True)
    return tot, items[:n]


def main():
    tag = sys.argv[1]
    args = sys.argv[2:]
    launches = None
    if "--launches" in args:
        i = args.index("--launches")
        launches = args[i + 1]
        args = args[:i] + args[i + 2:]
    # tag "tmp": scratch summaries outside the repo (iteration), else tracked under profiles/
    prof = "/tmp/prof" if tag == "tmp" else os.path.join(ROOT, "profiles")
    os.makedirs(prof, exist_ok=True)
    for rep in args:
        kern = os.path.basename(rep).replace(".ncu-rep", "").replace("prof_", "")
        out = [f"# ncu --set full --clock-control none capture of {kern} ({tag})", f"# source: {rep}", ""]
        recs = raw(rep)
        for d in recs:
            out.append(f"kernel: {d.get('Kernel Name', ('?',))[0]}")
            for k in KEYS:
                if k in d:
                    out.append(f"  {k:64s} {d[k][0]:>18s} {d[k][1]}")
            out.append("")
        tot, top = lines(rep)
        out.append(f"top source lines by warp-stall samples (total {tot}):")
        for w, loc, s in top:
            out.append(f"  {w:8d} {100 * w / max(tot, 1):5.1f}%  {loc:26s} {s}")
        with open(os.path.join(prof, f"{tag}_{kern}.txt"), "w") as fh:
            fh.write("\n".join(out) + "\n")
        if recs:
            d = recs[0]

            def mb(k):
                v, u = d[k]
                v = float(v.replace(",", ""))
                return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)

            js = {"kernel": kern, "tag": tag,
                  "dram_bytes_per_launch": mb("dram__bytes_read.sum") + mb("dram__bytes_write.sum"),
                  "duration_ms_ncu": float(d["gpu__time_duration.sum"][0].replace(",", "")) *
                  {"usecond": 1e-3, "us": 1e-3, "nsecond": 1e-6, "ns": 1e-6}.get(d["gpu__time_duration.sum"][1], 1.0),
                  "fp64_pipe_pct": float(d["sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"][0]),
                  "issue_active_pct": float(d["smsp__issue_active.avg.pct_of_peak_sustained_active"][0]),
                  "warps_active_pct": float(d["sm__warps_active.avg.pct_of_peak_sustained_active"][0]),
                  "l2_hit_pct": float(d["lts__t_sector_hit_rate.pct"][0]),
                  "note": "ncu --set full, cold-cache serialized replay; traffic = dram read + write bytes; "
                          "l2 bytes = lts__t_sectors x 32"}
            if "lts__t_sectors.sum" in d:
                js["lts_bytes_per_launch"] = 32.0 * float(d["lts__t_sectors.sum"][0].replace(",", ""))
                js["lts_gbs_ncu"] = js["lts_bytes_per_launch"] / (js["duration_ms_ncu"] * 1e-3) / 1e9
            js["dram_gbs_ncu"] = js["dram_bytes_per_launch"] / (js["duration_ms_ncu"] * 1e-3) / 1e9
            if "l1tex__t_sector_hit_rate.pct" in d:
                js["l1_hit_pct"] = float(d["l1tex__t_sector_hit_rate.pct"][0])
            with open(os.path.join(prof, f"{kern}_ncu.json"), "w") as fh:
                json.dump(js, fh, indent=1)
        print("wrote", kern)
    if launches:
        rows = list(csv.reader(open(launches)))
        hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
        h = rows[hi]
        ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
        d = defaultdict(list)
        for r in rows[hi + 1:]:
            if len(r) > vi:
                v = float(r[vi].replace(",", ""))
                v *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(r[ui], 1.0)
                d[r[ki].split("(")[0]].append(v)
        out = [f"# ncu --metrics gpu__time_duration.sum --clock-control none launch list ({tag})",
               "# cold-cache, serialised per-launch times: compare SHARES of the step, not absolutes", "",
               f"{'kernel':60s} {'n':>4s} {'mean_us':>10s} {'total_us':>11s}"]
        for k, v in sorted(d.items(), key=lambda x: -sum(x[1])):
            out.append(f"{k[:60]:60s} {len(v):4d} {sum(v) / len(v):10.1f} {sum(v):11.1f}")
        with open(os.path.join(prof, f"{tag}_launches.txt"), "w") as fh:
            fh.write("\n".join(out) + "\n")
        print("wrote launches")


if __name__ == "__main__":
    main()
