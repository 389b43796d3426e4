cd $GRAFT_REPO_ROOT
for c in vector+fifo "vector+bucket(d4)" near_far+fifo "near_far+bucket(d1)" filter+fifo "filter+bucket(d4)" slf+fifo "slf+bucket(d1)"; do
  l1=${c%%+*}; l2=${c#*+}
  timeout 60 python tools/repro.py rmat 16 $l1 "$l2" 10 1024 auto > gpurun_out/r9.log 2>&1 || { echo "FAIL $c rc=$?" >> gpurun_out/repro9.log; grep -A5 "EXC" gpurun_out/r9.log | cut -c1-300 >> gpurun_out/repro9.log; }
  echo "$c ok=$(grep -c True gpurun_out/r9.log) false=$(grep -c False gpurun_out/r9.log)" >> gpurun_out/repro9.log
done
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/pytest_gpu.log
timeout 600 python tools/tune.py --config c2 --grid fifo > gpurun_out/tune_c2_fifo2.log 2>&1
