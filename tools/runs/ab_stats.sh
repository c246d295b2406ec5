# A/B of assign_stats_kernel (grid-stride shared histograms) against the previous build
# (libsc_b200_oldkm.so), alternating on one box
O=$PWD/paper_1509_08863_b200/libsc_b200_oldkm.so
python tools/time_stability.py c2_sbm100k >/dev/null 2>&1
for i in 1 2 3; do
  echo "new c4 $(SC_KMEANS_TRACE=1 python tools/time_kmeans.py c4_sbm10m 1 16 2>&1 | grep 'restart 0')"
  echo "old c4 $(SC_B200_LIB=$O SC_KMEANS_TRACE=1 python tools/time_kmeans.py c4_sbm10m 1 16 2>&1 | grep 'restart 0')"
done
for i in 1 2 3; do
  echo "new c2 $(SC_STABILITY_TRACE=1 python tools/time_stability.py c2_sbm100k 2>&1 | grep k-means)"
  echo "old c2 $(SC_B200_LIB=$O SC_STABILITY_TRACE=1 python tools/time_stability.py c2_sbm100k 2>&1 | grep k-means)"
done
