cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/pytest_gpu.log
timeout 900 python tools/sweep.py c2 'l1=vector cap=512,1024,2048 l0=1,4 wb=4,8,16,0 hub=3072 groups=auto' > gpurun_out/sweep_wb.log 2>&1
