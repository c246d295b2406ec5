# stability scan on configs[2] with the fp32 screen threshold lowered (SC_KMEANS_SCREEN_MIN)
python tools/time_stability.py c2_sbm100k > /dev/null 2>&1
for m in 134217728 30000000 10000000 134217728 30000000 10000000; do
  echo "screen_min=$m"; SC_KMEANS_SCREEN_MIN=$m SC_STABILITY_TRACE=1 python tools/time_stability.py c2_sbm100k 2>&1 | grep -E "k-means|seconds" | cut -c1-150
done
