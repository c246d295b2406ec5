#!/bin/bash
# (1) column-chunk width vs the gathered table's L2 footprint on configs[3] (SELL kernel)
# (2) configs[4] on 1 GPU (SELL vs CSR) and the 8-rank grid emulation on the same box
o=gpurun_out/r02_chunk24.txt; : > $o
smi() { nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv,noheader >> $o; }
timeout 900 python -m pytest tests -m gpu -x -q -k "p2p or dist or partition or grid or emulated or rank or nccl" 2>&1 | tail -3 >> $o
smi
timeout 600 python tools/sweep_filter.py --workload c3_sbm1m --chunks 32,24,16,32 --reps 3 --tag sell >> $o 2>&1
smi
timeout 900 python tools/sweep_filter.py --workload c4_sbm10m --chunks 0 --reps 1 --tag c4_sell >> $o 2>&1
smi
SC_SELL=0 timeout 900 python tools/sweep_filter.py --workload c4_sbm10m --chunks 0 --reps 1 --tag c4_csr >> $o 2>&1
smi
timeout 1200 python tools/grid_emulate.py c4_sbm10m 8 >> $o 2>&1
smi
timeout 600 python tools/sweep_filter.py --workload c4_sbm10m --chunks 0 --reps 1 --tag c4_sell_again >> $o 2>&1
smi
cut -c1-300 $o
