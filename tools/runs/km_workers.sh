# sc_cluster phases on configs[3] with 4 / 5 / 10 k-means worker threads (SC_KMEANS_WORKERS)
o=gpurun_out/km_workers.txt; : > $o
for wk in 4 5 10 4 5 10; do
  echo "workers=$wk" >> $o
  SC_KMEANS_WORKERS=$wk python tools/time_cluster.py c3_sbm1m >> $o 2>&1
done
cat $o
