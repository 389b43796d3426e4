timeout 1300 python -m pytest tests -m gpu -x -q > gpurun_out/h_gputests.log 2>&1; echo "rc=$?" >> gpurun_out/h_gputests.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/h_smoke.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/h_bench_c2.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 --config c5 --no-cpu --no-g500 > gpurun_out/h_bench_c5.log 2>&1
timeout 900 python bench.py --steps 3 --warmup 3 --config c4 --no-cpu --no-g500 > gpurun_out/h_bench_c4.log 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 --config c3 --no-cpu --no-g500 > gpurun_out/h_bench_c3.log 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --config c1 --no-cpu --no-g500 > gpurun_out/h_bench_c1.log 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/h_bench_ref.log 2>&1
NCU="ncu --set full --cache-control none --clock-control none --import-source on -k regex:mlmq_persistent -s 3 -c 1"
timeout 900 $NCU -f -o gpurun_out/r2e_c5_k1 python tools/prof_run.py c5 --reps 4 > gpurun_out/h_ncu_c5.log 2>&1
