mkdir -p gpurun_out
AB_G=128,64 timeout 600 python scripts/exp/abbench_group.py base t1 e1 te1 abl15 te15 > gpurun_out/gq_abl2.log 2>&1
