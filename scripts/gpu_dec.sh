mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_decode_gpu.py -x -q > gpurun_out/t_dec.log 2>&1; echo "rc=$?" >> gpurun_out/t_dec.log
timeout 300 python scripts/kbench.py decode --iters 20 > gpurun_out/kb_dec.log 2>&1; echo "rc=$?" >> gpurun_out/kb_dec.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:kv_decode_kernel -c 1 -o gpurun_out/dec_mha -f python scripts/exp/one_decode.py 64 64 64 > gpurun_out/ncu_dec.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:kv_decode_kernel -c 1 -o gpurun_out/dec_gqa -f python scripts/exp/one_decode.py 64 8 64 >> gpurun_out/ncu_dec.log 2>&1
