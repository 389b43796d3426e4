cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_sharded.py -x -q -m gpu > gpurun_out/pytest_shard.log 2>&1; echo pytest=$? >> gpurun_out/pytest_shard.log
for P in 1 2 4 8; do timeout 300 python tools/shard_repro.py $P 20 >> gpurun_out/shard_s20.log 2>&1; done
