mkdir -p gpurun_out
QUAROT_LIB=$PWD/_variants/libquarot_ahigh.so timeout 600 python -m pytest tests/test_parity_gpu.py -q -x -k "s32_bit_exact" > gpurun_out/t_ahigh.log 2>&1; echo rc=$? >> gpurun_out/t_ahigh.log
for r in 1 2 3; do for v in new ahigh; do
  if [ $v = new ]; then L=$PWD/paper_2404_00456_b200/libquarot.so; else L=$PWD/_variants/libquarot_$v.so; fi
  echo "== $v"; QUAROT_LIB=$L timeout 300 python scripts/exp/ab_gemms.py 2>&1 | tail -1
done; done > gpurun_out/ab_ahigh.log 2>&1
true
