cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/selector
timeout 2400 python tools/selector_sweep.py gpurun_out/selector > gpurun_out/selector/sweep.log 2>&1; echo rc=$? >> gpurun_out/selector/sweep.log
