#!/bin/bash
# k-means tensor screen: wide register prefetch (d <= 128, 1 CTA/SM) -- parity + configs[4] timing
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "kmeans or cluster or stability" > gpurun_out/w_tests.log 2>&1; echo "tests_rc=$?" >> gpurun_out/w_tests.log
SC_KMEANS_TRACE=1 SC_TC_PROFILE=1 timeout 900 python tools/time_kmeans_wide.py c4_sbm10m 10 20 > gpurun_out/w_c4.log 2>&1; echo "rc=$?" >> gpurun_out/w_c4.log
tail -3 gpurun_out/w_tests.log; grep -v "tensor screen: " gpurun_out/w_c4.log | tail -12; grep "tensor screen" gpurun_out/w_c4.log | sort | uniq -c | head
timeout 600 python tools/time_cluster.py c3_sbm1m 3 > gpurun_out/w_c3cluster.log 2>&1; echo "rc=$?" >> gpurun_out/w_c3cluster.log
grep -v "^\[" gpurun_out/w_c3cluster.log | tail -4; grep "k-means\|kmeans" gpurun_out/w_c3cluster.log | tail -3
