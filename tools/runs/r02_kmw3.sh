python -m pytest tests -q -m gpu -x -k "kmeans or cluster or stability" 2>&1 | tail -2
python tools/time_cluster.py c3_sbm1m 3 2>&1 | grep -E "sc_cluster" | tail -2
python tools/time_stability.py 2>&1 | grep -oE '"seconds": [0-9.]+'
python tools/time_stability.py 2>&1 | grep -oE '"seconds": [0-9.]+'
