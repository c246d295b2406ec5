# k-means launch lists (ncu, cold cache, serialised) on configs[3] and configs[4] features
python tools/time_kmeans.py c3_sbm1m 1 30 > gpurun_out/km_c3_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"assign|check|member|plan|scatter|stats|d2_|seed|range|centroid|zero" \
    --csv --log-file gpurun_out/km_c3_launches.csv python tools/time_kmeans.py c3_sbm1m 1 30 > gpurun_out/km_c3_ncu.log 2>&1
SC_KMEANS_TRACE=1 python tools/time_kmeans.py c4_sbm10m 1 10 > gpurun_out/km_c4_plain.log 2>&1
