bash scripts/gpu_full_tests.sh
timeout 600 python bench.py > gpurun_out/bench_final.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_final.log
