timeout 900 ncu --set full --clock-control none --import-source on -k regex:"check_kernel" -s 20 -c 1 -o gpurun_out/r02_check_full \
  python tools/time_kmeans_pipe.py c3_sbm1m 1 100 > /dev/null 2>&1; echo "ncu rc=$?"
