cd $GRAFT_REPO_ROOT
timeout 600 python tools/sweep.py c1 'l1=vector cap=256 l2=bucket d=4,8 win=1 groups=148,592' > gpurun_out/sweep_c1g.log 2>&1
timeout 600 python tools/sweep.py c1 'l1=vector,filter cap=256,1024 l0=1,4 l2=fifo groups=148,592,auto' >> gpurun_out/sweep_c1g.log 2>&1
timeout 600 python tools/sweep.py c3 'l1=vector cap=256 l2=bucket d=8 win=1 groups=1184,auto reps=1' >> gpurun_out/sweep_c1g.log 2>&1
timeout 600 python tools/sweep.py c2 'l1=vector cap=1024 l0=1 hub=3072 groups=auto' >> gpurun_out/sweep_c1g.log 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/pytest_gpu.log
