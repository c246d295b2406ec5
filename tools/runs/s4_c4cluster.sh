#!/bin/bash
# configs[4] sc_cluster end to end with the phase split (1 rep) + restart split
mkdir -p gpurun_out
SC_KMEANS_TRACE=1 timeout 1200 python tools/time_cluster.py c4_sbm10m 2 > gpurun_out/c4cl.log 2>&1; echo "rc=$?" >> gpurun_out/c4cl.log
grep -v "^\[sc_kmeans\] iteration" gpurun_out/c4cl.log | grep -v "tensor screen" | tail -30
