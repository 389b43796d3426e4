set -x
for c in c2 c5 c4; do
  ck=--check; [ $c = c4 ] && ck=
  echo "== $c base"; python tools/prof_run.py $c --reps 5 $ck 2>&1 | grep -E "rep 4|best|oracle"
  echo "== $c dtok"; MLMQ_LIB=paper_2602_10080_b200/libmlmq_dtok.so python tools/prof_run.py $c --reps 5 $ck 2>&1 | grep -E "rep 4|best|oracle"
done
