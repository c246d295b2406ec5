# round 2: tensor screen chunk size experiment
for r in 1 2 3; do python tools/time_cluster.py c3_sbm1m 1 2>&1 | grep -E "sc_cluster"; done
K='regex:assign_tc'
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -s 100 -c 20 --csv --log-file gpurun_out/r02_tc_chunk.csv \
  env SC_CLUSTER_TRACE= python tools/time_cluster.py c3_sbm1m 1 > /dev/null 2>&1; echo "ncu rc=$?"
