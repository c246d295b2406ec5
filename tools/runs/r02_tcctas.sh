# round 2: tensor-screen grid (CTAs per SM) vs concurrency with the other restarts' kernels
for c in 3 2 1; do echo "SC_TC_CTAS=$c"; for r in 1 2; do SC_TC_CTAS=$c python tools/time_cluster.py c3_sbm1m 1 2>&1 | grep -E "sc_cluster"; done; done
for w in 2 4 8; do echo "SC_KMEANS_WORKERS=$w"; SC_KMEANS_WORKERS=$w python tools/time_cluster.py c3_sbm1m 1 2>&1 | grep -E "sc_cluster"; done
