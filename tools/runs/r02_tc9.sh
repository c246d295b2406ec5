# round 2: full ncu capture of the tensor screen v2 inside the configs[3] pipeline (iteration ~30)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:assign_tc_kernel -s 30 -c 1 -o gpurun_out/r02_km_tc_full3 \
  env SC_CLUSTER_TRACE= python tools/time_cluster.py c3_sbm1m 1 > gpurun_out/tcfull3.log 2>&1; echo "ncu rc=$?"
