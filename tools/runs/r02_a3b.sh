# round 2: exact-scan tile width (NC) for the screen's ambiguous points, configs[3] pipeline
for nc in 4 1; do echo "SC_KMEANS_NC=$nc"; SC_KMEANS_NC=$nc python tools/time_cluster.py c3_sbm1m 2 2>&1 | grep -E "sc_cluster|seconds"; done
K='regex:assign3'
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -s 100 -c 30 --csv --log-file gpurun_out/r02_a3_nc4.csv \
  env SC_CLUSTER_TRACE= python tools/time_cluster.py c3_sbm1m 1 > /dev/null 2>&1; echo "ncu rc=$?"
python -m pytest tests -q -m gpu -x -k "kmeans or cluster or stability" 2>&1 | tail -2
