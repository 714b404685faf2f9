timeout 300 python -m pytest tests/test_parity_gpu.py tests/test_transform_variants_gpu.py -q -k "11008 or full" > gpurun_out/t172.log 2>&1; echo rc=$? >> gpurun_out/t172.log
for r in 1 2; do for v in base new; do
 if [ $v = base ]; then L=$PWD/_variants/libquarot_base.so; else L=$PWD/paper_2404_00456_b200/libquarot.so; fi
 echo "== $v"; QUAROT_LIB=$L HQ_CASES=full:11008 python scripts/kbench.py hq --iters 20 2>&1 | grep "^full"
 QUAROT_LIB=$L HQ_CASES=full:11008 python scripts/kbench.py hq --iters 50 --tokens 16384 2>&1 | grep "^full"
done; done > gpurun_out/h172ab.log
