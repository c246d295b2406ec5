# round 2: steady-state Lloyd iteration launch list (configs[3] features, 1 restart, 100 iterations)
SC_KMEANS_TRACE=1 python tools/time_kmeans.py c3_sbm1m 1 100 > gpurun_out/km100.log 2>&1 || exit 1
K='regex:assign|group|check|member|plan|scatter|stats|finalize|centroid_prep|lo_|bound|hamerly|update'
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -s 500 -c 150 --csv --log-file gpurun_out/r02_km_steady_launches.csv \
  python tools/time_kmeans.py c3_sbm1m 1 100 > gpurun_out/kmncu.log 2>&1; echo "ncu rc=$?"
