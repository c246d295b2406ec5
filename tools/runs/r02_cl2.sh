# round 2: sc_cluster (configs[3]) Lloyd-phase launch list + per-iteration queue lengths
SC_KMEANS_TRACE=1 python tools/time_cluster.py c3_sbm1m 1 > gpurun_out/cl_trace.log 2>&1 || exit 1
K='regex:assign|group|check|member|plan|scatter|stats|finalize|centroid_prep'
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -s 600 -c 200 --csv --log-file gpurun_out/r02_cl_steady_launches.csv \
  env SC_CLUSTER_TRACE= python tools/time_cluster.py c3_sbm1m 1 > gpurun_out/clncu.log 2>&1; echo "ncu rc=$?"
