# A/B of the FULL K = 28672 quantizer: self-scheduled (default) vs producer warps (variant 4) vs round-2 head
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_transform_variants_gpu.py tests/test_glue_gpu.py -q -x -k "full or chain or 28672 or 11008 or 13b" > gpurun_out/t_hq6.log 2>&1; echo rc=$? >> gpurun_out/t_hq6.log
for r in 1 2; do
 echo "== head"; QUAROT_LIB=$PWD/_variants/libquarot_head.so VARIANTS=kperm,0 ROUNDS=3 timeout 300 python scripts/hqfull_ab.py 2>&1 | head -2
 echo "== new"; VARIANTS=kperm,0 ROUNDS=3 timeout 300 python scripts/hqfull_ab.py 2>&1 | head -4
 for v in head new; do
  if [ $v = new ]; then L=$PWD/paper_2404_00456_b200/libquarot.so; else L=$PWD/_variants/libquarot_$v.so; fi
  echo "== kb $v"; QUAROT_LIB=$L HQ_CASES=full:11008,full:13824,full:5120 timeout 300 python scripts/kbench.py hq --iters 20 2>&1 | grep "^full"
 done
done > gpurun_out/hq_ab6.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:hq_full28_wg -c 1 -o gpurun_out/hqwg_kperm6 -f python scripts/exp/one_hqfull.py 32768 28672 0 kperm > gpurun_out/ncu_hqwg5.log 2>&1
ncu -i gpurun_out/hqwg_kperm6.ncu-rep --page source --csv --print-source sass > gpurun_out/hqwg_kperm6_src.csv 2>/dev/null
true
