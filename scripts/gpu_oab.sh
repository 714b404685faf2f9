timeout 300 python -m pytest tests/test_glue_gpu.py tests/test_parity_gpu.py tests/test_shard_gpu.py -x -q > gpurun_out/t_res.log 2>&1; echo rc=$? >> gpurun_out/t_res.log
for v in base; do QUAROT_LIB=$PWD/_variants/libquarot_$v.so python scripts/exp/o_residual_ab.py > gpurun_out/oab_$v.log 2>&1; done
python scripts/exp/o_residual_ab.py > gpurun_out/oab_new.log 2>&1
for r in 1 2; do
QUAROT_LIB=$PWD/_variants/libquarot_base.so timeout 300 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/ab_base_$r.json 2>/dev/null
timeout 300 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/ab_new_$r.json 2>/dev/null
done
