for v in base hpt16; do
  if [ $v = base ]; then L=""; else L=_variants/libquarot_$v.so; fi
  echo "== $v"
  QUAROT_LIB=$L timeout 200 python scripts/kbench.py hq 2>&1 | grep "across"
  QUAROT_LIB=$L timeout 200 python -m pytest tests/test_parity_gpu.py -q -k across 2>&1 | tail -1
done
