#!/bin/bash
o=gpurun_out/r02_seedbatch2.txt; : > $o
for b in 1 0 1 0; do
  SC_KMEANS_SEED_BATCH=$b REPS=3 timeout 600 python tools/time_stability.py 2>&1 | cut -c1-120 | sed "s/^/batch$b /" >> $o
done
cat $o
