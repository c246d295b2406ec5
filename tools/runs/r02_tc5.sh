# round 2: full ncu capture of the k-means tensor screen (configs[3] features)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:assign_tc_kernel -s 2 -c 1 -o gpurun_out/r02_km_tc_full \
  python tools/time_kmeans.py c3_sbm1m 1 5 > gpurun_out/tcfull.log 2>&1; echo "ncu rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:assign_screen_kernel -s 2 -c 1 -o gpurun_out/r02_km_f32_full \
  env SC_KMEANS_TC=0 python tools/time_kmeans.py c3_sbm1m 1 5 > gpurun_out/f32full.log 2>&1; echo "ncu rc=$?"
