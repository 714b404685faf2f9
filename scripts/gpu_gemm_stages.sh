mkdir -p gpurun_out
for r in 1 2 3; do for v in base s2o4; do
  L=$PWD/_variants/libquarot_$v.so
  echo "== $v"; QUAROT_LIB=$L timeout 300 python scripts/exp/ab_gemms.py 2>&1 | tail -1
done; done > gpurun_out/ab_gemm_stages.log 2>&1
true
