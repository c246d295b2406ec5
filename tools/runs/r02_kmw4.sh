nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv
for r in 1 2 3; do python tools/time_stability.py 2>&1 | grep -oE '"seconds": [0-9.]+'; done
