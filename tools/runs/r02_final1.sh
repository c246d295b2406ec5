# round 2: bench line (configs[3]) + steady k-means launch list of the committed tensor screen
python bench.py > gpurun_out/r02_bench_c3.json 2> gpurun_out/r02_bench_c3.err; echo "bench rc=$?"
K='regex:assign|group|check|member|plan|scatter|stats|finalize|centroid_prep|amb_scan|tc_panel|tc_fix'
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -s 600 -c 300 --csv --log-file gpurun_out/r02_cl_steady_launches.csv \
  env SC_CLUSTER_TRACE= python tools/time_cluster.py c3_sbm1m 1 > gpurun_out/clncu.log 2>&1; echo "ncu rc=$?"
SC_KMEANS_TRACE=1 python tools/time_cluster.py c3_sbm1m 1 2>&1 | grep -E "ambiguous" | awk "{print \$4, \$6}" | awk '{r+=$1; a+=$2; n++} END {print n, "assignments, mean rescanned", r/n, "mean ambiguous", a/n}'
