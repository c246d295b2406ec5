#!/bin/bash
# moments on the SELL kernel (exact fixed-point sums): parity/determinism + timing vs CSR
o=gpurun_out/r02_mom_sell.txt; : > $o
timeout 1200 python -m pytest tests -m gpu -x -q -k "moments or lambda or cluster or stability or smoke or eigencount" 2>&1 | tail -4 >> $o
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv,noheader >> $o
timeout 600 python tools/time_moments.py c3_sbm1m 32 2>&1 | sed 's/^/sell /' >> $o
SC_SELL=0 timeout 600 python tools/time_moments.py c3_sbm1m 32 2>&1 | grep moments | sed 's/^/csr /' >> $o
SC_CLUSTER_TRACE=1 timeout 600 python tools/time_cluster.py c3_sbm1m >> $o 2>&1
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv,noheader >> $o
cat $o | cut -c1-300
# configs[4] 8-rank grid: chunk width of the 48-column rank blocks (48 = one 192-B-row chunk by
# default; 32 + 16 or 3 x 16 instead), SELL vs CSR in the ranks
for ch in 32 16; do
  SC_CHUNK=$ch timeout 900 python tools/grid_emulate.py c4_sbm10m 8 2>&1 | grep grid | sed "s/^/chunk$ch /" >> $o
  SC_SELL=0 SC_CHUNK=$ch timeout 900 python tools/grid_emulate.py c4_sbm10m 8 2>&1 | grep grid | sed "s/^/csr_chunk$ch /" >> $o
done
timeout 900 python tools/sweep_filter.py --workload c4_sbm10m --chunks 0 --reps 1 --tag c4_1gpu >> $o 2>&1
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv,noheader >> $o
cut -c1-300 $o | tail -8
