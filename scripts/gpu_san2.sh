mkdir -p gpurun_out
export SAN_M=300
timeout 600 python scripts/sanitize_run.py > gpurun_out/san_plain.log 2>&1; echo "rc=$?" >> gpurun_out/san_plain.log
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python scripts/sanitize_run.py > gpurun_out/san_memcheck.log 2>&1; echo "rc=$?" >> gpurun_out/san_memcheck.log
timeout 1200 compute-sanitizer --tool synccheck --print-limit 20 python scripts/sanitize_run.py > gpurun_out/san_synccheck.log 2>&1; echo "rc=$?" >> gpurun_out/san_synccheck.log
timeout 1500 compute-sanitizer --tool racecheck --racecheck-report analysis --print-limit 20 python scripts/sanitize_run.py > gpurun_out/san_racecheck.log 2>&1; echo "rc=$?" >> gpurun_out/san_racecheck.log
true
