# round 2: tensor screen with d = 96 (non-prefetch staging) and k = 200
SC_KMEANS_TRACE=1 python -m pytest tests -q -m gpu -x -k "kmeans_bit_exact" 2>&1 | grep -E "passed|failed|Error|tensor screen" | sort | uniq -c | head
