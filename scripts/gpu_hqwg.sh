mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:hq_full28_wg -c 1 -o gpurun_out/hqwg_kperm -f python scripts/exp/one_hqfull.py 32768 28672 0 kperm > gpurun_out/ncu_hqwg.log 2>&1
