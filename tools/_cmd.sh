cd $GRAFT_REPO_ROOT
for w in 32 64; do echo "want=$w" >> gpurun_out/sweep_own2.log; MLMQ_L1_WANT=$w timeout 600 python tools/sweep.py c2 'l1=vector cap=1024 l0=1 hub=3072 groups=auto reps=5' >> gpurun_out/sweep_own2.log 2>&1; done
MLMQ_L1_WANT=64 timeout 600 python tools/sweep.py c5 'l1=vector cap=1024 l0=1 hub=3072 groups=auto' >> gpurun_out/sweep_own2.log 2>&1
