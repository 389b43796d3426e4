cd $GRAFT_REPO_ROOT
timeout 600 python tools/sweep.py c2 'l1=vector cap=256,1024 l0=1,4 hub=3072 groups=auto' > gpurun_out/sweep_lb2.log 2>&1
timeout 600 python tools/sweep.py c1 'l1=vector cap=256 l2=bucket d=4 win=2 groups=148,592' >> gpurun_out/sweep_lb2.log 2>&1
timeout 600 python tools/sweep.py c3 'l1=vector cap=256 l2=bucket d=4 win=2 groups=1184 reps=1' >> gpurun_out/sweep_lb2.log 2>&1
