# round 2: every k-means kernel of one sc_cluster-feature restart (100 iterations), serialised
K='regex:assign|amb_scan|tc_|group_|member_|plan_members|scatter_any|check_kernel|d2_update|seed_select|range_sums|centroid_prep|row_to_centroid|absmax'
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -c 2500 --csv --log-file gpurun_out/r02_km_restart_launches.csv \
  python tools/time_kmeans_pipe.py c3_sbm1m 1 100 > gpurun_out/kmall.log 2>&1; echo "ncu rc=$?"
