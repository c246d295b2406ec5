# round 2: tensor screen v2 (fp32 epilogue, prefetched rows): parity, timings, launch lists
python -m pytest tests -q -m gpu -x -k "kmeans or cluster" 2>&1 | tail -3
SC_KMEANS_TRACE=1 python tools/time_kmeans.py c3_sbm1m 1 5 2>&1 | grep -E "CTAs|seconds" | tail -2
for tc in 1 0; do echo "SC_KMEANS_TC=$tc"; SC_KMEANS_TC=$tc python tools/time_cluster.py c3_sbm1m 3 2>&1 | grep -E "sc_cluster|seconds"; done
K='regex:assign|group|check|member|plan|scatter|stats|finalize|centroid_prep'
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -s 600 -c 200 --csv --log-file gpurun_out/r02_cl_steady_launches.csv \
  env SC_CLUSTER_TRACE= python tools/time_cluster.py c3_sbm1m 1 > gpurun_out/clncu.log 2>&1; echo "ncu rc=$?"
SC_TC_PROFILE=1 python tools/time_cluster.py c3_sbm1m 1 2>&1 | grep -E "cycles per CTA" | tail -1
