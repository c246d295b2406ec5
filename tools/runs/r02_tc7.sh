# round 2: k-means tensor screen, full ncu capture + launch list after the grid fix
python tools/time_kmeans.py c3_sbm1m 1 5 > gpurun_out/tcplain.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:assign_tc_kernel -s 2 -c 1 -o gpurun_out/r02_km_tc_full2 \
  python tools/time_kmeans.py c3_sbm1m 1 5 > gpurun_out/tcfull.log 2>&1; echo "ncu rc=$?"
K='regex:assign|group|check|member|plan|scatter|stats|finalize|centroid_prep'
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -c 200 --csv --log-file gpurun_out/r02_km_tc_launches.csv \
  python tools/time_kmeans.py c3_sbm1m 1 5 > gpurun_out/tcncu.log 2>&1; echo "ncu rc=$?"
