mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_transform_variants_gpu.py tests/test_shard_gpu.py -q -x -k "full or 28672 or 11008 or kperm" > gpurun_out/t_ph.log 2>&1; echo rc=$? >> gpurun_out/t_ph.log
for r in 1 2 3; do for v in new plow; do
  if [ $v = new ]; then L=$PWD/paper_2404_00456_b200/libquarot.so; else L=$PWD/_variants/libquarot_$v.so; fi
  echo "== $v"; QUAROT_LIB=$L VARIANTS=kperm ROUNDS=3 timeout 300 python scripts/hqfull_ab.py 2>&1 | head -1
  QUAROT_LIB=$L HQ_CASES=full:11008 timeout 300 python scripts/kbench.py hq --iters 20 --tokens 131072 2>&1 | grep "^full"
  QUAROT_LIB=$L HQ_CASES=full:11008 timeout 300 python scripts/kbench.py hq --iters 50 --tokens 16384 2>&1 | grep "^full"
done; done > gpurun_out/ab_ph.log 2>&1
true
