# round 2: tensor-core k-means screen after the grouping / epilogue / staging fixes
o=gpurun_out/r02_tc2.txt; : > $o
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "kmeans or cluster" >> $o 2>&1
echo "pytest rc=$?" >> $o
for i in 1 2; do
timeout 300 python tools/time_kmeans.py c3_sbm1m 1 20 >> $o 2>&1
SC_KMEANS_TC=0 timeout 300 python tools/time_kmeans.py c3_sbm1m 1 20 >> $o 2>&1
done
timeout 300 python tools/time_kmeans.py c3_sbm1m 10 100 >> $o 2>&1
SC_KMEANS_TC=0 timeout 300 python tools/time_kmeans.py c3_sbm1m 10 100 >> $o 2>&1
python tools/time_kmeans.py c3_sbm1m 1 5 > gpurun_out/tcplain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/r02_km_launches.csv \
  python tools/time_kmeans.py c3_sbm1m 1 5 > gpurun_out/tcncu.log 2>&1; echo "ncu rc=$?" >> $o
