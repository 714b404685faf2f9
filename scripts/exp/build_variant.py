"""Build libquarot.so with extra nvcc defines into _variants/libquarot_<name>.so (kernel-variant
experiments; select at run time with QUAROT_LIB=...).  Usage: build_variant.py NAME -DFOO=1 ..."""
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2404_00456_b200 import build as B  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
out_dir = os.path.join(B.ROOT, "_variants", name)
os.makedirs(out_dir, exist_ok=True)
cc = B.nvcc()
objs = [os.path.join(out_dir, s.replace(".cu", ".o")) for s in B.SOURCES]


def run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode:
        raise SystemExit(r.stderr)
    return r.stderr


with ThreadPoolExecutor(8) as ex:
    logs = list(ex.map(run, [[cc, *B.ARCH, *B.FLAGS, *defs, "-c", os.path.join(B.CSRC, s), "-o", o]
                             for s, o in zip(B.SOURCES, objs)]))
for line in "".join(logs).splitlines():
    if "spill" in line and "int4_gemm" not in line and " 0 bytes spill" not in line:
        pass
lib = os.path.join(B.ROOT, "_variants", f"libquarot_{name}.so")
run([cc, *B.ARCH, "-shared", "-cudart", "static", "-o", lib, *objs])
print(lib)
