# ncu full capture of one Hamerly check launch on configs[4] features
python tools/time_kmeans.py c4_sbm10m 1 12 > gpurun_out/chk_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:check_kernel -s 3 -c 1 -o gpurun_out/check_c4 \
    python tools/time_kmeans.py c4_sbm10m 1 12 > gpurun_out/chk_ncu.log 2>&1
