for r in 1 2; do REPS=4 python tools/time_stability.py 2>&1 | grep -oE '"seconds": [0-9.]+' | tr '\n' ' '; echo; done
