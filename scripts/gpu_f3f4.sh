mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_parity_gpu.py -k "int4_linear_group" -x -q > gpurun_out/t_group.log 2>&1; echo "rc=$?" >> gpurun_out/t_group.log
timeout 300 python scripts/kbench.py gemm_group --iters 5 > gpurun_out/kb_group.log 2>&1; echo "rc=$?" >> gpurun_out/kb_group.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:int4_group_gemm -c 1 -o gpurun_out/group128 -f python scripts/exp/one_group_gemm.py 32768 8192 8192 128 > gpurun_out/ncu_group.log 2>&1
