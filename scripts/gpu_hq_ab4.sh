# A/B of the FULL K = 28672 quantizer: current tree vs _variants/libquarot_head.so (+ parity tests)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_transform_variants_gpu.py tests/test_glue_gpu.py -q -x -k "full or chain or 28672" > gpurun_out/t_hq.log 2>&1; echo rc=$? >> gpurun_out/t_hq.log
for r in 1 2; do for v in head new; do
 if [ $v = new ]; then L=$PWD/paper_2404_00456_b200/libquarot.so; else L=$PWD/_variants/libquarot_$v.so; fi
 echo "== $v"; QUAROT_LIB=$L VARIANTS=kperm,0 ROUNDS=3 timeout 300 python scripts/hqfull_ab.py 2>&1 | head -2
done; done > gpurun_out/hq_ab4.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:hq_full28_wg -c 1 -o gpurun_out/hqwg_kperm4 -f python scripts/exp/one_hqfull.py 32768 28672 0 kperm > gpurun_out/ncu_hqwg4.log 2>&1
ncu -i gpurun_out/hqwg_kperm4.ncu-rep --page raw --csv > gpurun_out/hqwg_kperm4_raw.csv 2>/dev/null
ncu -i gpurun_out/hqwg_kperm4.ncu-rep --page source --csv --print-source sass > gpurun_out/hqwg_kperm4_src.csv 2>/dev/null
true
