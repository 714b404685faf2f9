# SwiGLU fast division (gate/up GEMM) and 172 producer back-off: new vs r3prev; glue + 11008 parity
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_glue_gpu.py tests/test_parity_gpu.py -q -x -k "swiglu or chain or 11008 or fused or glue" > gpurun_out/t_ab9.log 2>&1; echo rc=$? >> gpurun_out/t_ab9.log
for r in 1 2 3; do for v in new r3prev; do
  if [ $v = new ]; then L=$PWD/paper_2404_00456_b200/libquarot.so; else L=$PWD/_variants/libquarot_$v.so; fi
  echo "== $v"; QUAROT_LIB=$L timeout 300 python scripts/exp/ab_gateup.py 2>&1 | tail -1
done; done > gpurun_out/ab9_gateup.log 2>&1
for r in 1 2; do for v in new p172spin p172sleep r3prev; do
  if [ $v = new ]; then L=$PWD/paper_2404_00456_b200/libquarot.so; else L=$PWD/_variants/libquarot_$v.so; fi
  echo "== $v"; QUAROT_LIB=$L HQ_CASES=full:11008 timeout 300 python scripts/kbench.py hq --iters 20 --tokens 131072 2>&1 | grep "^full"
  QUAROT_LIB=$L HQ_CASES=full:11008 timeout 300 python scripts/kbench.py hq --iters 50 --tokens 16384 2>&1 | grep "^full"
done; done > gpurun_out/ab9_172.log 2>&1
true
