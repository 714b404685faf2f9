mkdir -p gpurun_out
for r in 1 2 3; do for v in new kv5; do
  if [ $v = new ]; then L=$PWD/paper_2404_00456_b200/libquarot.so; else L=$PWD/_variants/libquarot_$v.so; fi
  echo "== $v"; QUAROT_LIB=$L timeout 300 python scripts/kbench.py kv --iters 20 2>&1 | grep "^kv"
done; done > gpurun_out/kv_ab.log 2>&1
true
