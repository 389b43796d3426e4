cd $GRAFT_REPO_ROOT
for P in 2 4 8; do timeout 600 python bench.py --config c2 --parts $P --steps 3 --warmup 2 --no-cpu > gpurun_out/bench_c2_p$P.log 2>&1; done
timeout 1500 python bench.py --config c4 --parts 8 --steps 2 --warmup 1 --no-cpu > gpurun_out/bench_c4_p8.log 2>&1
