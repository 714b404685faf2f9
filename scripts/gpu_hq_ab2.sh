mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_parity_gpu.py tests/test_transform_variants_gpu.py tests/test_glue_gpu.py -q -x -k "full or chain or 11008 or 13b" > gpurun_out/t_hq.log 2>&1; echo rc=$? >> gpurun_out/t_hq.log
for r in 1 2; do for v in head new; do
 if [ $v = head ]; then L=$PWD/_variants/libquarot_head.so; else L=$PWD/paper_2404_00456_b200/libquarot.so; fi
 echo "== $v"; QUAROT_LIB=$L HQ_CASES=full:28672,full:11008,full:13824,full:5120 python scripts/kbench.py hq --iters 20 2>&1 | grep "^full"
 QUAROT_LIB=$L VARIANTS=kperm ROUNDS=3 python scripts/hqfull_ab.py 2>&1 | head -2
done; done > gpurun_out/hq_ab2.log 2>&1
