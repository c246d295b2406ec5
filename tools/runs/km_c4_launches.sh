# k-means launch list on configs[4] features (1 restart, 3 Lloyd iterations)
python tools/time_kmeans.py c4_sbm10m 1 3 > gpurun_out/km_c4_plain2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"assign|check|member|plan|scatter|stats|d2_|seed|range|centroid|zero|row_to" \
    --csv --log-file gpurun_out/km_c4_launches.csv python tools/time_kmeans.py c4_sbm10m 1 3 > gpurun_out/km_c4_ncu.log 2>&1
