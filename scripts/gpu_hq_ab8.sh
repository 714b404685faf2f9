# FULL-28 with H_2 in the MMA (new) vs the previous commit (r3prev); parity tests first
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_transform_variants_gpu.py tests/test_glue_gpu.py -q -x -k "full or 28672 or chain" > gpurun_out/t_hq8.log 2>&1; echo rc=$? >> gpurun_out/t_hq8.log
for r in 1 2 3; do for v in new r3prev; do
  if [ $v = new ]; then L=$PWD/paper_2404_00456_b200/libquarot.so; else L=$PWD/_variants/libquarot_$v.so; fi
  echo "== $v"; QUAROT_LIB=$L VARIANTS=kperm,0 ROUNDS=3 timeout 300 python scripts/hqfull_ab.py 2>&1 | head -4
done; done > gpurun_out/hq_ab8.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:hq_full28_wg -c 1 -o gpurun_out/hqwg_kperm8 -f python scripts/exp/one_hqfull.py 32768 28672 0 kperm > gpurun_out/ncu_hqwg8.log 2>&1
ncu -i gpurun_out/hqwg_kperm8.ncu-rep --page source --csv --print-source sass > gpurun_out/hqwg_kperm8_src.csv 2>/dev/null
true
