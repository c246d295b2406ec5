# stability scan on configs[2]: Hamerly-check threshold (SC_KMEANS_PRUNE_MIN) with the screen threshold at 3e7
python tools/time_stability.py c2_sbm100k > /dev/null 2>&1
for m in 134217728 30000000 134217728 30000000; do
  echo "prune_min=$m"; SC_KMEANS_PRUNE_MIN=$m SC_STABILITY_TRACE=1 python tools/time_stability.py c2_sbm100k 2>&1 | grep -E "k-means|seconds" | cut -c1-150
done
python tools/time_cluster.py c3_sbm1m | cut -c1-160
