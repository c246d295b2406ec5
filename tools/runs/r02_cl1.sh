# round 2: sc_cluster phase breakdown on configs[3], tensor screen on / off
for tc in 1 0; do echo "SC_KMEANS_TC=$tc"; SC_KMEANS_TC=$tc SC_KMEANS_TRACE=1 python tools/time_cluster.py c3_sbm1m 3 2>&1 | grep -vE "iteration|CTAs"; done
