mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:int4_gemm_kernel -s 1 -c 1 -o gpurun_out/gemm_gu -f python scripts/exp/one_gemm.py 32768 57344 8192 2 > gpurun_out/ncu_gemm.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:int4_gemm_kernel -s 1 -c 1 -o gpurun_out/gemm_o -f python scripts/exp/one_gemm.py 32768 8192 8192 2 >> gpurun_out/ncu_gemm.log 2>&1
