mkdir -p gpurun_out
for r in 1 2 3; do for v in new wgua wgbo32 wgbo160; do
  if [ $v = new ]; then L=$PWD/paper_2404_00456_b200/libquarot.so; else L=$PWD/_variants/libquarot_$v.so; fi
  echo "== $v"; QUAROT_LIB=$L VARIANTS=kperm ROUNDS=3 timeout 300 python scripts/hqfull_ab.py 2>&1 | head -1
done; done > gpurun_out/wg_micro.log 2>&1
true
