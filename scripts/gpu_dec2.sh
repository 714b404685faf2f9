mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_decode_gpu.py -q -x > gpurun_out/t_dec2.log 2>&1; echo rc=$? >> gpurun_out/t_dec2.log
for r in 1 2; do timeout 300 python scripts/kbench.py decode --iters 20 2>&1 | grep -E "^decode_" | sed -E 's/"ms_append_decode": [0-9.]+, //; s/"gbs_decode": [0-9.]+, //'; done > gpurun_out/dec2.log 2>&1
true
