for v in base o4s3 spin o4s3spin; do
  if [ $v = base ]; then L=""; else L=_variants/libquarot_$v.so; fi
  echo "== $v"
  QUAROT_LIB=$L timeout 120 python scripts/dbg_gemm_full.py 2>&1 | grep -c "bad=0"
  QUAROT_LIB=$L timeout 200 python scripts/kbench.py ksweep gemm 2>&1 | grep -v '^{"gemm' | grep -v '"mode": 1' | cut -c1-150
done
