# round 2: moments determinism test; stability scan split (configs[2]) with the tensor screen on / off
python -m pytest tests -q -m gpu -x -k "deterministic" 2>&1 | tail -2
for tc in 1 0; do echo "SC_KMEANS_TC=$tc"; for r in 1 2; do SC_KMEANS_TC=$tc SC_STABILITY_TRACE=1 python tools/time_stability.py 2>&1 | grep -E "sc_stability\]|seconds" | cut -c1-160; done; done
