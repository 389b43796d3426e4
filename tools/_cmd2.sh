for c in c2 c5; do for lib in base cold cold2 base; do
  L=paper_2602_10080_b200/libmlmq_$lib.so; [ $lib = base ] && L=paper_2602_10080_b200/libmlmq.so
  echo "== $lib $c"; MLMQ_LIB=$L timeout 600 python tools/prof_run.py $c --reps 7 --golden 2>&1 | tail -2
done; done > gpurun_out/cold.log 2>&1
for lib in cold2 base; do
  L=paper_2602_10080_b200/libmlmq_$lib.so; [ $lib = base ] && L=paper_2602_10080_b200/libmlmq.so
  echo "== $lib c3"; MLMQ_LIB=$L timeout 600 python tools/prof_run.py c3 --reps 3 2>&1 | tail -1
  echo "== $lib c4"; MLMQ_LIB=$L timeout 900 python tools/prof_run.py c4 --reps 4 --golden 2>&1 | tail -2
done >> gpurun_out/cold.log 2>&1
MLMQ_LIB=paper_2602_10080_b200/libmlmq_cold2.so timeout 600 python -m pytest tests/test_gpu_errors_and_big.py -q -k "overflow or watchdog" > gpurun_out/cold_err.log 2>&1
