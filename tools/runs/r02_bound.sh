# round 2: bound-only pruning in the screened path: parity + timings
python -m pytest tests -q -m gpu -x -k "kmeans or cluster or stability" 2>&1 | tail -2
for b in 1 0; do echo "SC_KMEANS_BOUND=$b"; SC_KMEANS_BOUND=$b python tools/time_cluster.py c3_sbm1m 3 2>&1 | grep -E "sc_cluster|info" | tail -2 | cut -c1-200; done
SC_KMEANS_TRACE=1 python tools/time_cluster.py c3_sbm1m 1 2>&1 | grep -E "ambiguous" | awk "{print \$4, \$6}" | awk '{r+=$1; a+=$2; n++} END {print n, "assignments, mean rescanned", r/n, "mean ambiguous", a/n}'
