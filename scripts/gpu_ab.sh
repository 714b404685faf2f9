mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_parity_gpu.py tests/test_glue_gpu.py -x -q -k "gemm or linear or chain_small or residual or swiglu" > gpurun_out/t_gemm.log 2>&1; echo "rc=$?" >> gpurun_out/t_gemm.log
for r in 1 2; do
QUAROT_LIB=$PWD/_variants/libquarot_base.so timeout 300 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/ab_base_$r.json 2>/dev/null
timeout 300 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/ab_new_$r.json 2>/dev/null
done
