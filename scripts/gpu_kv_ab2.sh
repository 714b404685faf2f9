mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_glue_gpu.py tests/test_parity_gpu.py tests/test_decode_gpu.py -q -x -k "rope or kv or fused or chain or decode" > gpurun_out/t_kv2.log 2>&1; echo rc=$? >> gpurun_out/t_kv2.log
for r in 1 2 3; do for v in new kvhead; do
  if [ $v = new ]; then L=$PWD/paper_2404_00456_b200/libquarot.so; else L=$PWD/_variants/libquarot_$v.so; fi
  echo "== $v"; QUAROT_LIB=$L timeout 300 python scripts/exp/kv_shapes.py 2>&1 | cat
done; done > gpurun_out/kv_ab2.log 2>&1
true
