mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench_chain.json 2> gpurun_out/bench_chain.err
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_chain.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
echo launches rc=$?
# one full capture of each kernel family in one chain step at 32768 tokens (launch order: see launches csv)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'int4_gemm|hq_|kv_quant|kv_tc|rope' -c 10 -o gpurun_out/chain_full python bench.py --profile-steps 1 --tokens 32768 > gpurun_out/ncu_full.log 2>&1
echo full rc=$?
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:'int4_gemm|hq_|kv_quant|kv_tc|rope' -c 10 --csv --log-file gpurun_out/traffic_chain.csv python bench.py --profile-steps 1 > /dev/null 2>&1
echo traffic rc=$?
