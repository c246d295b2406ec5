# round 2: configs[4] sc_cluster phases, tensor screen on / off
for tc in 1 0; do echo "SC_KMEANS_TC=$tc"; SC_KMEANS_TC=$tc SC_KMEANS_TRACE=1 timeout 1200 python tools/time_cluster.py c4_sbm10m 1 2>&1 | grep -E "sc_cluster|seconds|CTAs|restart 9"; done
