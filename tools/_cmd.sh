cd $GRAFT_REPO_ROOT
for c in vector+fifo "vector+bucket(d1)" "near_far+bucket(d4)" "filter+bucket(d4)" "slf+bucket(d1)" slf+fifo; do
  l1=${c%%+*}; l2=${c#*+}
  timeout 60 python tools/repro.py rmat 16 $l1 "$l2" 4 1024 auto > gpurun_out/r9.log 2>&1 || { echo "FAIL $c rc=$?" >> gpurun_out/repro13.log; grep -A5 "EXC" gpurun_out/r9.log | cut -c1-300 >> gpurun_out/repro13.log; }
  echo "$c ok=$(grep -c True gpurun_out/r9.log) false=$(grep -c False gpurun_out/r9.log)" >> gpurun_out/repro13.log
  timeout 60 python tools/repro.py grid 256 $l1 "$l2" 4 1024 auto > gpurun_out/r9.log 2>&1 || { echo "FAIL grid $c rc=$?" >> gpurun_out/repro13.log; grep -A5 "EXC" gpurun_out/r9.log | cut -c1-300 >> gpurun_out/repro13.log; }
  echo "grid $c ok=$(grep -c True gpurun_out/r9.log) false=$(grep -c False gpurun_out/r9.log)" >> gpurun_out/repro13.log
done
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/pytest_gpu.log
timeout 300 python tools/sweep.py c2 'l1=vector cap=1024 l0=1 hub=3072' > gpurun_out/sweep_c1d.log 2>&1
timeout 900 python tools/sweep.py c1 'l1=vector cap=256 l2=bucket d=2,4,8 win=1,2 groups=148,592,auto' >> gpurun_out/sweep_c1d.log 2>&1
timeout 900 python tools/sweep.py c3 'l1=vector cap=256 l2=bucket d=4,16 win=2 groups=1184,auto reps=1' >> gpurun_out/sweep_c1d.log 2>&1
