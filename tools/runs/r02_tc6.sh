# round 2: k-means tensor screen after the occupancy / exact-distance changes
python -m pytest tests -q -m gpu -x -k "kmeans or cluster" 2>&1 | tail -3
for tc in 1 0; do SC_KMEANS_TC=$tc SC_KMEANS_TRACE=1 python tools/time_kmeans.py c3_sbm1m 1 5 2>&1 | grep -E "CTAs|seconds" | tail -2; done
for tc in 1 0; do SC_KMEANS_TC=$tc python tools/time_kmeans.py c3_sbm1m 10 100; done
K='regex:assign|group|check|member|plan|scatter|stats|finalize|centroid_prep'
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -c 200 --csv --log-file gpurun_out/r02_km_tc_launches.csv \
  python tools/time_kmeans.py c3_sbm1m 1 5 > gpurun_out/tcncu.log 2>&1; echo "ncu rc=$?"
