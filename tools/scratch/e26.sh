run() { echo "== $*"; python tools/prof_run.py "$@" 2>&1 | grep -E "rep 4|best|oracle|L2 persist"; }
L=paper_2602_10080_b200
for c in c2 c5 c4; do
  r=5; [ $c = c4 ] && r=3
  run $c --reps $r
  MLMQ_LIB=$L/libmlmq_hint1.so run $c --reps $r
  MLMQ_LIB=$L/libmlmq_hint2.so run $c --reps $r
  MLMQ_L2PERSIST=1 run $c --reps $r
  MLMQ_L2PERSIST=0.5 run $c --reps $r
  MLMQ_L2PERSIST=1 MLMQ_LIB=$L/libmlmq_hint2.so run $c --reps $r --check
done
