# round 2: exact scan of the ambiguous points with 16-point tiles
python -m pytest tests -q -m gpu -x -k "kmeans or cluster or stability" 2>&1 | tail -2
python tools/time_cluster.py c3_sbm1m 3 2>&1 | grep -E "sc_cluster|seconds"
K='regex:assign3'
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -s 100 -c 30 --csv --log-file gpurun_out/r02_a3_amb.csv \
  env SC_CLUSTER_TRACE= python tools/time_cluster.py c3_sbm1m 1 > /dev/null 2>&1; echo "ncu rc=$?"
