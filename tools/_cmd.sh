cd $GRAFT_REPO_ROOT
timeout 900 python tools/sweep.py c2 'l1=vector cap=1024 l0=1,4 hub=3072,4096,6144,8192 groups=1184,auto' > gpurun_out/sweep_hub.log 2>&1
timeout 1200 python tools/sweep.py c3 'l1=vector,filter cap=1024 l2=fifo,bucket d=1,8 reps=1' > gpurun_out/sweep_c3.log 2>&1
