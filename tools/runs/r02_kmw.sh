# round 2: k-means restart workers (concurrent streams) on the configs[3] pipeline, 4 reps each
for w in 4 8 10 4 8 10; do echo "SC_KMEANS_WORKERS=$w"; SC_KMEANS_WORKERS=$w python tools/time_cluster.py c3_sbm1m 4 2>&1 | grep -E "sc_cluster" | tail -3 | awk '{print $(NF-1)}' | tr '\n' ' '; echo; done
