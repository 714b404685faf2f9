# Round-2 final evidence (second session): GPU tests, smoke, bench lines, launch list, DRAM traffic, kernel bench
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --config 7b --steps 50 > gpurun_out/bench7b.json 2> gpurun_out/bench7b.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_chain.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-peak-probe > /dev/null 2>&1
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:'int4_gemm|hq_|kv_quant|kv_tc' -c 9 --csv --log-file gpurun_out/traffic_chain.csv python bench.py --profile-steps 1 > /dev/null 2>&1
timeout 600 python scripts/kbench.py gemm hq kv --iters 10 > gpurun_out/kbench_main.log 2>&1
echo done
