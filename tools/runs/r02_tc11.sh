# round 2: full ncu captures of the tensor screen and the exact scan of its ambiguous points (configs[3] pipeline)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"assign_tc_kernel|assign3_kernel|tc_panel|tc_fix|group_plan" -s 150 -c 5 -o gpurun_out/r02_km_tc_full5 \
  env SC_CLUSTER_TRACE= python tools/time_cluster.py c3_sbm1m 1 > gpurun_out/tcfull5.log 2>&1; echo "ncu rc=$?"
