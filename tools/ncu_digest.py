"""Digest of one ncu --set full capture exported by tools/gpu_prof.sh
(<tag>_raw.csv + <tag>_sass.csv): duration, DRAM bytes, pipe / issue
utilisation, stall reasons per issue and the executed SASS mix per TMA box
step.  Prints the text committed under profiles/."""
import collections
import csv
import sys

tag = sys.argv[1]
steps_key = sys.argv[2] if len(sys.argv) > 2 else "UTMALDG"
rows = list(csv.reader(open(f"gpurun_out/{tag}_raw.csv")))
h, u, v = rows[0], rows[1], rows[2]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "smsp__warps_eligible.avg.per_cycle_active"]
for w in want:
    if w in h:
        i = h.index(w)
        print(f"{w:80s} {v[i]} {u[i]}")
print("\n# stall reasons (warps per issue-active cycle)")
for i, n in enumerate(h):
    if n.startswith("smsp__average_warps_issue_stalled_") and n.endswith("_per_issue_active.ratio"):
        try:
            x = float(v[i])
        except ValueError:
            continue
        if x >= 0.02:
            print(f"  {n[34:-23]:28s} {x:.3f}")
srows = list(csv.reader(open(f"gpurun_out/{tag}_sass.csv")))
hi = [i for i, r in enumerate(srows) if "Source" in r][0]
sh = srows[hi]
iS, iE = sh.index("Source"), sh.index("Instructions Executed")
ops = collections.Counter()
for r in srows[hi + 1:]:
    try:
        n = int(r[iE].replace(",", ""))
    except (ValueError, IndexError):
        continue
    t = r[iS].split()
    if not t:
        continue
    op = t[1] if t[0].startswith("@") else t[0]
    ops[op.split(".")[0]] += n
tot = sum(ops.values())
steps = ops.get(steps_key, 1)
print(f"\n# executed SASS (warp-level): {tot} total, {steps} {steps_key} (one per box step), "
      f"{tot / steps:.1f} per box")
for k, n in ops.most_common(24):
    print(f"  {k:10s} {n:12d} {n / tot * 100:5.1f}%  {n / steps:7.1f}/box")
