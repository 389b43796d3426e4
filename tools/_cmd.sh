cd $GRAFT_REPO_ROOT
for c in c2 c5 c1 c3; do timeout 900 python bench.py --config $c --steps 10 --warmup 3 --cpu-budget-s 10 > gpurun_out/bench_${c}_final.log 2>&1; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2_final.csv python bench.py --steps 2 --warmup 1 --no-cpu > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mlmq_persistent -s 3 -c 1 -o gpurun_out/prof_c2_final python tools/one_solve.py c2 vector fifo 1 512 5 > gpurun_out/ncu_full_final.log 2>&1
