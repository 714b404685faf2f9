mkdir -p gpurun_out
export SAN_M=300
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python scripts/sanitize_run.py > gpurun_out/san_memcheck.log 2>&1; echo "rc=$?" >> gpurun_out/san_memcheck.log
timeout 900 compute-sanitizer --tool racecheck --racecheck-report analysis --print-limit 20 python scripts/sanitize_run.py > gpurun_out/san_racecheck.log 2>&1; echo "rc=$?" >> gpurun_out/san_racecheck.log
timeout 900 compute-sanitizer --tool synccheck --print-limit 20 python scripts/sanitize_run.py > gpurun_out/san_synccheck.log 2>&1; echo "rc=$?" >> gpurun_out/san_synccheck.log
timeout 600 python scripts/hqfull_ab.py > gpurun_out/hqfull_ab.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:hq_full28_wg -c 1 -o gpurun_out/hqwg -f python scripts/exp/one_hqfull.py 32768 28672 > gpurun_out/ncu_hqwg.log 2>&1
