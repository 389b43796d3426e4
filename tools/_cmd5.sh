timeout 600 python tools/scratch/sweep_heavy.py c5 0.01 0.02 0.04 0.02 > gpurun_out/hd.log 2>&1
timeout 300 python tools/scratch/sweep_heavy.py c2 16 24 32 24 >> gpurun_out/hd.log 2>&1
timeout 900 python tools/scratch/sweep_heavy.py c4 12 16 24 32 48 24 >> gpurun_out/hd.log 2>&1
