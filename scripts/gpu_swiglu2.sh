mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_glue_gpu.py tests/test_shard_gpu.py tests/test_streams_gpu.py -q -x > gpurun_out/t_sw2.log 2>&1; echo rc=$? >> gpurun_out/t_sw2.log
for r in 1 2 3; do for v in new gemmhead; do
  if [ $v = new ]; then L=$PWD/paper_2404_00456_b200/libquarot.so; else L=$PWD/_variants/libquarot_$v.so; fi
  echo "== $v"; QUAROT_LIB=$L timeout 300 python scripts/exp/ab_gateup.py 2>&1 | tail -1
done; done > gpurun_out/ab_sw2.log 2>&1
true
