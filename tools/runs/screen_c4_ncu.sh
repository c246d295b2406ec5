# ncu full capture of one k-means screen launch on configs[4] features
python tools/time_kmeans.py c4_sbm10m 1 3 > gpurun_out/scr_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:assign_screen -s 2 -c 1 -o gpurun_out/screen_c4 \
    python tools/time_kmeans.py c4_sbm10m 1 3 > gpurun_out/scr_ncu.log 2>&1
