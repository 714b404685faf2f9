timeout 400 python -m pytest tests/test_parity_gpu.py tests/test_shard_gpu.py tests/test_transform_variants_gpu.py tests/test_fullsize_gpu.py -q -x -k "full or kperm or 28672 or shard or step" > gpurun_out/t_park.log 2>&1; echo rc=$? >> gpurun_out/t_park.log
VARIANTS=4,kperm,0,4,kperm,0 ROUNDS=3 timeout 300 python scripts/hqfull_ab.py > gpurun_out/park_ab.log 2>&1
