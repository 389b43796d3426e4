timeout 900 python tools/scratch/sweep_groups.py c4 1776 2220 2400 2663 > gpurun_out/grp4.log 2>&1
timeout 600 python tools/scratch/sweep_groups.py c5 2220 2663 2959 >> gpurun_out/grp4.log 2>&1
