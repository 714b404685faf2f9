mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:kv_tc -c 1 -o gpurun_out/kv_rope -f python scripts/exp/one_kv.py 32768 rope > gpurun_out/ncu_kv.log 2>&1
ncu -i gpurun_out/kv_rope.ncu-rep --page source --csv --print-source sass > gpurun_out/kv_rope_src.csv 2>/dev/null
timeout 600 ncu --set full --import-source on --clock-control none -k regex:hq_full172 -c 1 -o gpurun_out/h172 -f python scripts/exp/one_hqfull.py 32768 11008 > gpurun_out/ncu_h172.log 2>&1
ncu -i gpurun_out/h172.ncu-rep --page source --csv --print-source sass > gpurun_out/h172_src.csv 2>/dev/null
true
