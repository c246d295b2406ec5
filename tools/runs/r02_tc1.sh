# round 2: tcgen05 probe + the tensor-core k-means screen (parity + timing)
o=gpurun_out/r02_tc1.txt; : > $o
timeout 120 ./tools/tcp >> $o 2>&1; echo "tcp rc=$?" >> $o
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "kmeans or cluster or stability" >> $o 2>&1
echo "pytest rc=$?" >> $o
SC_KMEANS_TRACE=1 timeout 300 python tools/time_kmeans.py c3_sbm1m 1 20 >> $o 2>gpurun_out/tc_trace.txt; echo "tc rc=$?" >> $o
SC_KMEANS_TC=0 timeout 300 python tools/time_kmeans.py c3_sbm1m 1 20 >> $o 2>&1
timeout 300 python tools/time_kmeans.py c3_sbm1m 10 100 >> $o 2>&1
SC_KMEANS_TC=0 timeout 300 python tools/time_kmeans.py c3_sbm1m 10 100 >> $o 2>&1
tail -30 gpurun_out/tc_trace.txt >> $o
