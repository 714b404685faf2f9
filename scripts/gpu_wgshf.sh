mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_shard_gpu.py -q -x -k "full or 28672 or kperm" > gpurun_out/t_shf.log 2>&1; echo rc=$? >> gpurun_out/t_shf.log
for r in 1 2 3 4; do for v in new wgprev; do
  if [ $v = new ]; then L=$PWD/paper_2404_00456_b200/libquarot.so; else L=$PWD/_variants/libquarot_$v.so; fi
  echo "== $v"; QUAROT_LIB=$L VARIANTS=kperm ROUNDS=3 timeout 300 python scripts/hqfull_ab.py 2>&1 | head -1
done; done > gpurun_out/ab_shf.log 2>&1
true
