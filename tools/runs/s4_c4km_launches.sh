#!/bin/bash
# launch list (gpu__time_duration) of configs[4] k-means: 1 restart x 6 Lloyd iterations
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c4km_launches.csv \
  python tools/time_kmeans.py c4_sbm10m 1 6 > gpurun_out/c4km_ncu.log 2>&1; echo "rc=$?" >> gpurun_out/c4km_ncu.log
tail -3 gpurun_out/c4km_ncu.log; wc -l gpurun_out/c4km_launches.csv
