# round 2: tensor screen v3 (panels + dynamic chunks): full capture + unfiltered steady launch list
timeout 900 ncu --set full --clock-control none --import-source on -k regex:assign_tc_kernel -s 30 -c 1 -o gpurun_out/r02_km_tc_full4 \
  env SC_CLUSTER_TRACE= python tools/time_cluster.py c3_sbm1m 1 > gpurun_out/tcfull4.log 2>&1; echo "ncu rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 2500 -c 300 --csv --log-file gpurun_out/r02_cl_all_launches.csv \
  env SC_CLUSTER_TRACE= python tools/time_cluster.py c3_sbm1m 1 > gpurun_out/clncu2.log 2>&1; echo "ncu rc=$?"
