cd $GRAFT_REPO_ROOT
for dbg in 1 0; do
for c in vector+fifo "vector+bucket(d1)" "vector+bucket(d4)" near_far+fifo "near_far+bucket(d1)" "near_far+bucket(d4)" filter+fifo "filter+bucket(d1)" "filter+bucket(d4)" slf+fifo "slf+bucket(d1)" "slf+bucket(d4)"; do
  l1=${c%%+*}; l2=${c#*+}
  MLMQ_DEBUG=$dbg timeout 60 python tools/repro.py rmat 16 $l1 "$l2" 20 1024 auto > gpurun_out/r8.log 2>&1 || { echo "FAIL dbg=$dbg $c rc=$?" >> gpurun_out/repro8.log; grep -A14 "stuck\|EXC" gpurun_out/r8.log | cut -c1-300 >> gpurun_out/repro8.log; }
  echo "dbg=$dbg $c ok=$(grep -c True gpurun_out/r8.log) false=$(grep -c False gpurun_out/r8.log)" >> gpurun_out/repro8.log
done
done
