for r in 1 2; do for v in 0 1; do
  echo "== vtxpack=$v"; MLMQ_VTXPACK=$v MLMQ_LIB=paper_2602_10080_b200/libmlmq_vtx.so timeout 300 python tools/prof_run.py c2 --reps 8 --golden 2>&1 | tail -2
done; done > gpurun_out/vtx.log 2>&1
MLMQ_VTXPACK=1 MLMQ_LIB=paper_2602_10080_b200/libmlmq_vtx.so timeout 300 python tools/prof_run.py c1 --reps 3 --check >> gpurun_out/vtx.log 2>&1
