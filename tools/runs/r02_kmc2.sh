# round 2: one stability-sized k-means problem (configs[2] features, k = 20, 5 restarts), trace
SC_KMEANS_TRACE=1 python tools/km_c2_probe.py 2>&1 | grep -E "restart|iters" | head -12
