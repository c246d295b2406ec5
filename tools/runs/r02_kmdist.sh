SC_KMEANS_TRACE=1 python -m pytest tests -q -s -m gpu -x -k "dist_kmeans_emulated" 2>&1 | grep -E "passed|failed|Error|assert|tensor screen" | sort | uniq -c | head -20
