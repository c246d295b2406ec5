# round 2: 10 restart workers by default: configs[3] pipeline, stability scan, configs[4] pipeline
python tools/time_cluster.py c3_sbm1m 3 2>&1 | grep -E "sc_cluster" | tail -2
for w in 10 4; do SC_KMEANS_WORKERS=$w python tools/time_stability.py 2>&1 | grep -oE '"seconds": [0-9.]+'; done
for w in 10 4; do echo "c4 workers $w"; SC_KMEANS_WORKERS=$w timeout 900 python tools/time_cluster.py c4_sbm10m 1 2>&1 | grep -E "sc_cluster"; done
