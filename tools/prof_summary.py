"""Summarise an ncu launch list (+ optional `--set full` capture) into the
text files committed under profiles/.

  python tools/prof_summary.py gpurun_out/<tag>_launches.csv [gpurun_out/<tag>_prof.ncu-rep] > profiles/<name>.txt

Launch list: per-kernel launch count, mean / min device time and share of
the summed time (ncu serialises launches and runs them cold, so compare
shares, not absolutes).  Full capture: duration, DRAM bytes (the roofline
`traffic` figure), throughput percentages, occupancy, registers and the
executed-instruction mix from the SASS source page.
"""
from __future__ import annotations

import collections
import csv
import io
import subprocess
import sys


def launches(path: str) -> None:
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    h = rows[0]
    ik, iv, iu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    ig, ib = h.index("Grid Size"), h.index("Block Size")
    per = collections.OrderedDict()
    for r in rows[1:]:
        name = r[ik].split("(")[0].replace("void ", "")[:70]
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3}.get(r[iu], 1e-3)
        t = float(r[iv].replace(",", "")) * scale
        per.setdefault((name, r[ig], r[ib]), []).append(t)
    tot = sum(sum(v) for v in per.values())
    print(f"# launch list: {path}")
    print(f"# {sum(len(v) for v in per.values())} launches, {tot:.1f} us summed device time")
    print(f"{'kernel':72s} {'grid':>14s} {'block':>12s} {'n':>4s} {'mean_us':>9s} {'min_us':>9s} {'share':>6s}")
    for (name, g, b), v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
        print(f"{name:72s} {g:>14s} {b:>12s} {len(v):4d} {sum(v)/len(v):9.2f} {min(v):9.2f} "
              f"{sum(v)/tot*100:5.1f}%")


def full(path: str) -> None:
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        print("# (no raw page)")
        return
    h, units, vals = rows[0], rows[1], rows[2:]
    want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
            "launch__grid_size", "launch__block_size", "launch__occupancy_limit_registers",
            "lts__t_sector_hit_rate.pct", "sm__cycles_elapsed.avg.per_second",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]
    print(f"\n# full capture: {path}")
    for v in vals:
        for w in want:
            if w in h:
                i = h.index(w)
                print(f"{w:60s} {v[i]:>20s} {units[i]}")
        print()
    src = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(src)))
    hdr = next((r for r in rows if "Source" in r and "Instructions Executed" in r), None)
    if not hdr:
        return
    iS, iE = hdr.index("Source"), hdr.index("Instructions Executed")
    iW = hdr.index("Warp Stall Sampling (All Samples)")
    mix, stall, tot = collections.Counter(), collections.Counter(), 0
    for r in rows[rows.index(hdr) + 1:]:
        if len(r) <= iE or not r[iE].isdigit():
            continue
        toks = r[iS].split()
        if not toks:
            continue
        op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
        op = op.split(".")[0]
        n = int(r[iE])
        mix[op] += n
        tot += n
        stall[op] += int(r[iW] or 0)
    print(f"# executed SASS instruction mix (warp-level), total {tot}")
    for op, n in mix.most_common(24):
        print(f"{op:10s} {n:12d} {n/tot*100:5.1f}%   stall samples {stall[op]}")


if __name__ == "__main__":
    launches(sys.argv[1])
    if len(sys.argv) > 2:
        full(sys.argv[2])
