"""Top SASS lines of an ncu report by warp-stall samples.  python scripts/ncu_top.py rep [n]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hh = rows[1]
iS, iE, iW, iA = hh.index("Source"), hh.index("Instructions Executed"), hh.index("Warp Stall Sampling (All Samples)"), hh.index("Address")
iN = hh.index("Warp Stall Sampling (Not-issued Samples)")
data = [r for r in rows[2:] if len(r) > iW]
print("total samples", sum(int(r[iW] or 0) for r in data))
for r in sorted(data, key=lambda r: -int(r[iW] or 0))[:n]:
    print(r[iA][-5:], r[iW], r[iN], r[iE], r[iS][:100])
