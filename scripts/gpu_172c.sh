mkdir -p gpurun_out
for r in 1 2 3; do for v in new lds_vol; do
  if [ $v = new ]; then L=$PWD/paper_2404_00456_b200/libquarot.so; else L=$PWD/_variants/libquarot_$v.so; fi
  echo "== $v"; QUAROT_LIB=$L HQ_CASES=full:11008 timeout 300 python scripts/kbench.py hq --iters 20 --tokens 131072 2>&1 | grep "^full"
  QUAROT_LIB=$L HQ_CASES=full:11008 timeout 300 python scripts/kbench.py hq --iters 50 --tokens 16384 2>&1 | grep "^full"
done; done > gpurun_out/ab_172c.log 2>&1
true
