mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:int4_group_gemm -c 1 -o gpurun_out/group128 python scripts/exp/one_group_gemm.py 32768 8192 8192 128 > gpurun_out/ncu_group.log 2>&1
echo rc=$? >> gpurun_out/ncu_group.log
