# steady-state k-means launch list on configs[4] features (1 restart, 16 iterations; the
# summary keeps the launches of the last iterations)
python tools/time_kmeans.py c4_sbm10m 1 16 > gpurun_out/km_c4s_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"assign|check|member|plan|scatter|stats|zero|centroid" \
    --csv --log-file gpurun_out/km_c4s_launches.csv python tools/time_kmeans.py c4_sbm10m 1 16 > gpurun_out/km_c4s_ncu.log 2>&1
