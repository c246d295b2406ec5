SC_KMEANS_TRACE=1 python -m pytest tests -q -s -m gpu -x -k "kmeans_bit_exact and (30000 or 20000-200)" 2>&1 | grep -E "passed|failed|tensor screen" | sort | uniq -c | head
