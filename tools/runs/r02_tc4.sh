# round 2: k-means launch lists of the Lloyd phase, tensor screen vs fp32 screen (configs[3] features, 1 restart, 5 iterations)
K='regex:assign|group|check|member|plan|scatter|stats|finalize|centroid_prep'
python tools/time_kmeans.py c3_sbm1m 1 5 > gpurun_out/tcplain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -c 200 --csv --log-file gpurun_out/r02_km_tc_launches.csv \
  python tools/time_kmeans.py c3_sbm1m 1 5 > gpurun_out/tcncu.log 2>&1; echo "ncu rc=$?"
SC_KMEANS_TC=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -c 200 --csv --log-file gpurun_out/r02_km_f32_launches.csv \
  python tools/time_kmeans.py c3_sbm1m 1 5 > gpurun_out/tcncu2.log 2>&1; echo "ncu2 rc=$?"
