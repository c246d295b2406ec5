#!/bin/bash
# column-group count of the 8-rank decomposition (configs[3] and configs[4]), same box as a 1-GPU pass
o=gpurun_out/r02_grid_cg.txt; : > $o
smi() { nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv,noheader >> $o; }
smi
timeout 600 python tools/sweep_filter.py --workload c3_sbm1m --chunks 0 --reps 3 --tag c3_1gpu >> $o 2>&1
timeout 900 python tools/grid_emulate.py c3_sbm1m 8 1,2,4,8 >> $o 2>&1
smi
timeout 900 python tools/sweep_filter.py --workload c4_sbm10m --chunks 0 --reps 1 --tag c4_1gpu >> $o 2>&1
timeout 2400 python tools/grid_emulate.py c4_sbm10m 8 4,8 >> $o 2>&1
smi
cut -c1-330 $o
