#!/bin/bash
# split-row (hub) kernel: gathers in flight per lane (SC_HUB_U) and blocks per SM, Chung-Lu
o=gpurun_out/r02_hub.txt; : > $o
smi() { nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv,noheader >> $o; }
smi
for lib in libsc_b200.so libsc_b200_hub8.so libsc_b200_hub4.so; do
  for bps in 8 4 2; do
    SC_HUB_BPS=$bps SC_B200_LIB=paper_1509_08863_b200/$lib timeout 300 python tools/sweep_filter.py --workload x_chunglu1m --chunks 32 --reps 2 --tag ${lib}_bps$bps >> $o 2>&1
  done
done
timeout 300 python tools/sweep_filter.py --workload c3_sbm1m --chunks 32 --reps 2 --tag c3 >> $o 2>&1
smi
cut -c1-200 $o
