mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_transform_variants_gpu.py tests/test_a8w8_gpu.py -q -x -k "heads" > gpurun_out/t_hh.log 2>&1; echo rc=$? >> gpurun_out/t_hh.log
for r in 1 2 3; do for v in new hhlow; do
  if [ $v = new ]; then L=$PWD/paper_2404_00456_b200/libquarot.so; else L=$PWD/_variants/libquarot_$v.so; fi
  echo "== $v"; QUAROT_LIB=$L HQ_CASES=across_heads:8192,across_heads:4096 timeout 300 python scripts/kbench.py hq --iters 20 --tokens 131072 2>&1 | grep "^across"
  QUAROT_LIB=$L HQ_CASES=across_heads:4096 timeout 300 python scripts/kbench.py hq --iters 50 --tokens 16384 2>&1 | grep "^across"
done; done > gpurun_out/ab_hh.log 2>&1
true
