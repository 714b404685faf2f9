for i in $(seq 1 15); do timeout 120 python -m pytest tests/test_glue_gpu.py -x -q -k "test_linear_residual" 2>&1 | tail -1; done > gpurun_out/dbg_res2.log
for i in 1 2 3 4 5; do python scripts/exp/dbg_res.py; done >> gpurun_out/dbg_res2.log 2>&1
