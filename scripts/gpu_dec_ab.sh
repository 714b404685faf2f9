mkdir -p gpurun_out
for r in 1 2; do for v in new dec2 dec8 dec16; do
  if [ $v = new ]; then L=$PWD/paper_2404_00456_b200/libquarot.so; else L=$PWD/_variants/libquarot_$v.so; fi
  echo "== $v"; QUAROT_LIB=$L timeout 300 python scripts/kbench.py decode --iters 20 2>&1 | grep -E "b16|b64" | sed -E 's/"ms_append_decode": [0-9.]+, //'
done; done > gpurun_out/dec_ab.log 2>&1
true
