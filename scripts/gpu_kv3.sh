mkdir -p gpurun_out
python -c "import torch; torch.zeros(1, device='cuda')"
for cfg in "37 8 64 1" "3 8 0 0"; do
  timeout 60 python scripts/exp/kv_hang.py $cfg >> gpurun_out/kv_hang.log 2>&1 || echo "FAIL/TIMEOUT $cfg" >> gpurun_out/kv_hang.log
done
if grep -q FAIL gpurun_out/kv_hang.log; then exit 0; fi
timeout 600 python -m pytest tests/test_glue_gpu.py tests/test_parity_gpu.py tests/test_decode_gpu.py -q -x -k "rope or kv or fused or chain or decode" > gpurun_out/t_kv2.log 2>&1; echo rc=$? >> gpurun_out/t_kv2.log
for r in 1 2; do for v in new kvhead; do
  if [ $v = new ]; then L=$PWD/paper_2404_00456_b200/libquarot.so; else L=$PWD/_variants/libquarot_$v.so; fi
  echo "== $v"; QUAROT_LIB=$L timeout 200 python scripts/exp/kv_shapes.py 2>&1 | cat
done; done > gpurun_out/kv_ab2.log 2>&1
true
