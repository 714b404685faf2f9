mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_transform_variants_gpu.py tests/test_a8w8_gpu.py -q -x -k "13824 or 5120 or 640 or 13b" > gpurun_out/t_small.log 2>&1; echo rc=$? >> gpurun_out/t_small.log
for r in 1 2 3; do for v in new smlow; do
  if [ $v = new ]; then L=$PWD/paper_2404_00456_b200/libquarot.so; else L=$PWD/_variants/libquarot_$v.so; fi
  echo "== $v"; QUAROT_LIB=$L HQ_CASES=full:13824,full:5120 timeout 300 python scripts/kbench.py hq --iters 20 --tokens 131072 2>&1 | grep "^full"
done; done > gpurun_out/ab_small.log 2>&1
true
