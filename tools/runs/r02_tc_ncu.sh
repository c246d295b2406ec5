#!/bin/bash
# ncu --set full of the tcgen05 k-means screen (assign_tc_kernel) inside sc_cluster on configs[3]
mkdir -p gpurun_out
python tools/time_cluster.py c3_sbm1m 1 > gpurun_out/tcn_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:assign_tc_kernel -s 20 -c 2 -o gpurun_out/tc_full \
    python tools/time_cluster.py c3_sbm1m 1 > gpurun_out/tcn_ncu.log 2>&1
echo "rc=$?"; tail -3 gpurun_out/tcn_ncu.log
