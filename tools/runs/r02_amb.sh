# round 2: per-iteration rescanned / ambiguous counts in the configs[3] pipeline, tensor screen on and off
for tc in 1 0; do echo "SC_KMEANS_TC=$tc"; SC_KMEANS_TC=$tc SC_KMEANS_TRACE=1 python tools/time_cluster.py c3_sbm1m 1 2>&1 | grep -E "ambiguous" | awk "{print \$4, \$6}" | sort -n | awk '{r+=$1; a+=$2; n++} END {print n, "assignments, mean rescanned", r/n, "mean ambiguous", a/n}'; done
