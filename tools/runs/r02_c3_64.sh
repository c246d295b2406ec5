#!/bin/bash
o=gpurun_out/r02_c3_64.txt; : > $o
timeout 900 python -m pytest tests -m gpu -x -q -k "moments or lambda or eigencount or hub or star or split or chung" 2>&1 | tail -2 >> $o
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv,noheader >> $o
timeout 600 python tools/sweep_filter.py --workload c3_sbm1m --chunks 32,64,32,64 --reps 3 --tag c3 >> $o 2>&1
timeout 600 python tools/sweep_filter.py --workload x_chunglu1m --chunks 32,64 --reps 2 --tag cl >> $o 2>&1
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv,noheader >> $o
cut -c1-200 $o
