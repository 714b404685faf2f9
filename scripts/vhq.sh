for v in base p1w8; do
  if [ $v = base ]; then L=""; else L=_variants/libquarot_$v.so; fi
  echo "== $v"
  QUAROT_LIB=$L timeout 200 python scripts/kbench.py hq 2>&1 | grep "full 28672"
done
