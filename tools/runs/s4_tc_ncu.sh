#!/bin/bash
# ncu --set full of the two-tile tensor screen (assign_tc_kernel<32,1,256>) on configs[4] features
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:assign_tc -s 1 -c 1 -o gpurun_out/tc_pair_c4 \
  python tools/time_kmeans.py c4_sbm10m 1 3 > gpurun_out/tc_ncu.log 2>&1; echo "rc=$?" >> gpurun_out/tc_ncu.log
tail -3 gpurun_out/tc_ncu.log; ls -la gpurun_out/*.ncu-rep
