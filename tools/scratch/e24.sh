run() { echo "== $*"; python tools/prof_run.py "$@" 2>&1 | grep -E "rep 4|best|oracle"; }
for h in 0 10 25 50 100; do run c1 --reps 5 --check --set heavy_delta=$h; done
for h in 16 20 28; do run c2 --reps 5 --set heavy_delta=$h; done
for hm in 4 16 64; do run c2 --reps 5 --set heavy_delta=24 heavy_min_edges=$hm; done
for h in 0.01 0.03; do run c5 --reps 3 --set heavy_delta=$h; done
for h in 25 50; do run c3 --reps 2 --set heavy_delta=$h cfg.l2_type=fifo; done
