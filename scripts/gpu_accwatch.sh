mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_glue_gpu.py tests/test_streams_gpu.py tests/test_fullsize_gpu.py -q -x -k "gemm or linear or chain or s32 or swiglu or residual or graph" > gpurun_out/t_aw.log 2>&1; echo rc=$? >> gpurun_out/t_aw.log
for r in 1 2 3; do for v in new gemmhead; do
  if [ $v = new ]; then L=$PWD/paper_2404_00456_b200/libquarot.so; else L=$PWD/_variants/libquarot_$v.so; fi
  echo "== $v"; QUAROT_LIB=$L timeout 300 python scripts/exp/ab_gemms.py 2>&1 | tail -1
done; done > gpurun_out/ab_aw.log 2>&1
for v in new gemmhead; do
  if [ $v = new ]; then L=$PWD/paper_2404_00456_b200/libquarot.so; else L=$PWD/_variants/libquarot_$v.so; fi
  echo "== $v"; QUAROT_LIB=$L timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['clocks'])"
done >> gpurun_out/ab_aw.log 2>&1
true
