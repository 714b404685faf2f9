mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_parity_gpu.py tests/test_transform_variants_gpu.py tests/test_glue_gpu.py -q -x -k "full or chain or 11008 or 13b" > gpurun_out/t_hq.log 2>&1; echo rc=$? >> gpurun_out/t_hq.log
for r in 1 2; do for v in head new bo32 bo160; do
 if [ $v = new ]; then L=$PWD/paper_2404_00456_b200/libquarot.so; else L=$PWD/_variants/libquarot_$v.so; fi
 echo "== $v"; QUAROT_LIB=$L HQ_CASES=full:28672,full:11008 python scripts/kbench.py hq --iters 20 2>&1 | grep "^full"
 QUAROT_LIB=$L VARIANTS=kperm ROUNDS=3 python scripts/hqfull_ab.py 2>&1 | head -1
done; done > gpurun_out/hq_ab3.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:hq_full28_wg -c 1 -o gpurun_out/hqwg_kperm2 -f python scripts/exp/one_hqfull.py 32768 28672 0 kperm > gpurun_out/ncu_hqwg2.log 2>&1
