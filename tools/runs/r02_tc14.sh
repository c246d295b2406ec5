python -m pytest tests -q -m gpu -x -k "kmeans or cluster or stability" 2>&1 | tail -2
SC_TC_PROFILE=1 python tools/time_cluster.py c3_sbm1m 1 2>&1 | grep -E "cycles per CTA|sc_cluster" | tail -2
