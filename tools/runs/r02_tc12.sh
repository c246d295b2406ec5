# round 2: full ncu capture of the tensor screen (two-chain epilogue) inside the configs[3] pipeline
timeout 900 ncu --set full --clock-control none --import-source on -k regex:assign_tc_kernel -s 30 -c 1 -o gpurun_out/r02_km_tc_full6 \
  env SC_CLUSTER_TRACE= python tools/time_cluster.py c3_sbm1m 1 > gpurun_out/tcfull6.log 2>&1; echo "ncu rc=$?"
