# round 2: full ncu capture of the exact scan of the screen's ambiguous points (configs[3] pipeline)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"assign3_kernel" -s 100 -c 1 -o gpurun_out/r02_km_a3_full \
  env SC_CLUSTER_TRACE= python tools/time_cluster.py c3_sbm1m 1 > gpurun_out/a3full.log 2>&1; echo "ncu rc=$?"
