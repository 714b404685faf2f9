"""Per-kernel SASS instruction-class counts of libquarot.so (cuobjdump -sass): the evidence that
the hot kernels run on tcgen05 (UTCIMMA / UTCHMMA), TMA (UTMALDG / UTMASTG / UBLKCP) and TMEM
(LDTM / STTM).  python scripts/sass_summary.py [libquarot.so] > profiles/rNN_sass_summary.txt"""
import collections
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2404_00456_b200/libquarot.so"
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
CLASSES = ["UTCIMMA", "UTCHMMA", "UTCQMMA", "UTMALDG", "UTMASTG", "UBLKCP", "LDTM", "STTM", "UTCBAR",
           "HMMA", "IMMA", "FADD2", "FFMA2", "FMUL2", "SYNCS", "USETMAXREG"]
kern, counts = None, collections.OrderedDict()
for line in out.splitlines():
    m = re.match(r"\s+Function : (\S+)", line)
    if m:
        kern = m.group(1)
        counts[kern] = collections.Counter()
        continue
    if kern is None:
        continue
    m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_]+)", line)
    if m:
        op = m.group(2)
        for c in CLASSES:
            if op.startswith(c):
                counts[kern][c] += 1
        counts[kern]["total"] += 1


def demangle(names):
    r = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.splitlines()
    return r if len(r) == len(names) else names


names = list(counts)
pretty = demangle(names)
print(f"# SASS instruction classes per kernel of {lib} (static counts, cuobjdump -sass)")
print(f"{'kernel':70s} " + " ".join(f"{c:>8s}" for c in CLASSES + ["total"]))
for n, p in zip(names, pretty):
    c = counts[n]
    p = re.sub(r"\(.*", "", p)[:70]
    print(f"{p:70s} " + " ".join(f"{c[k]:8d}" for k in CLASSES + ["total"]))
