"""Digest an ncu report: key throughput numbers, stall reasons, per-opcode executed counts.
python scripts/ncu_digest.py report.ncu-rep [units]   (units = rows for per-unit counts)"""
import collections, csv, io, subprocess, sys
rep = sys.argv[1]
units = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
h, v = r[0], r[2]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "sm__cycles_elapsed.avg.per_second",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed"]
for k, x in zip(h, v):
    if k in want:
        print(f"{k:70s} {x}")
for k, x in zip(h, v):
    if "average_warps_issue_stalled" in k and k.endswith("per_issue_active.ratio"):
        try:
            if float(x) > 0.05:
                print(f"  stall {k.split('stalled_')[1].split('_per')[0]:24s} {x}")
        except ValueError:
            pass
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hh = rows[1]
iS, iE, iW = hh.index("Source"), hh.index("Instructions Executed"), hh.index("Warp Stall Sampling (All Samples)")
cnt, st = collections.Counter(), collections.Counter()
tot = 0
for row in rows[2:]:
    try:
        n = int(row[iE])
    except (ValueError, IndexError):
        continue
    parts = row[iS].split()
    if not parts:
        continue
    op = parts[1] if parts[0].startswith("@") and len(parts) > 1 else parts[0]
    op = op.split(".")[0]
    cnt[op] += n
    st[op] += int(row[iW] or 0)
    tot += n
print(f"instructions executed: {tot}  per unit: {tot / units:.1f}")
for op, n in cnt.most_common(24):
    print(f"  {op:10s} {n / units:9.1f}  stall-samples {st[op]}")
