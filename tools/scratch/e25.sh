echo "== profile c2"; MLMQ_DEBUG=1 MLMQ_LIB=paper_2602_10080_b200/libmlmq_hprof.so python tools/prof_run.py c2 --reps 3 2>&1 | grep -E "mlmq debug\] |rep 2|best" | grep -v "warp \|wait states\|phase" | head -12
echo "== profile c5"; MLMQ_DEBUG=1 MLMQ_LIB=paper_2602_10080_b200/libmlmq_hprof.so python tools/prof_run.py c2 --reps 2 --set heavy_delta=0 2>&1 | grep -E "mlmq debug\] |best" | grep -v "warp \|wait states" | head -6
ncu --set full --cache-control none --clock-control none --import-source on -k regex:mlmq_persistent --launch-skip 3 --launch-count 1 -o gpurun_out/r2s_c2_k1 -f python tools/prof_run.py c2 --reps 4 > gpurun_out/r2s_ncu.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2s_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-g500 > gpurun_out/r2s_launch_bench.log 2>&1
echo done
