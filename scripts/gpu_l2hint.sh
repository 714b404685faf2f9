mkdir -p gpurun_out
for r in 1 2 3; do for v in new l2a l2b; do
  if [ $v = new ]; then L=$PWD/paper_2404_00456_b200/libquarot.so; else L=$PWD/_variants/libquarot_$v.so; fi
  echo "== $v"; QUAROT_LIB=$L timeout 300 python scripts/exp/ab_gemms.py 2>&1 | tail -1
done; done > gpurun_out/ab_l2.log 2>&1
for v in new l2a l2b; do
  if [ $v = new ]; then L=$PWD/paper_2404_00456_b200/libquarot.so; else L=$PWD/_variants/libquarot_$v.so; fi
  echo "== $v" >> gpurun_out/ab_l2.log
  QUAROT_LIB=$L timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:int4_gemm -c 1 --csv python scripts/exp/one_gemm.py 131072 8192 28672 1 2>/dev/null | grep -E "dram__|gpu__time" | awk -F'","' '{print $(NF-2), $(NF-1), $NF}' >> gpurun_out/ab_l2.log
done
true
