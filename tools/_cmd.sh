cd $GRAFT_REPO_ROOT
timeout 600 python tools/e2e_breakdown.py c2 > gpurun_out/e2e.log 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c2_r1b.log 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/pytest_gpu.log
