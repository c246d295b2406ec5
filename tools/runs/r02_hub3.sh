#!/bin/bash
o=gpurun_out/r02_hub3.txt; : > $o
for lib in libsc_b200.so libsc_b200_hc256.so libsc_b200.so libsc_b200_hc256.so; do
  SC_B200_LIB=paper_1509_08863_b200/$lib timeout 300 python tools/sweep_filter.py --workload x_chunglu1m --chunks 32 --reps 2 --tag ${lib} >> $o 2>&1
done
timeout 300 python tools/sweep_filter.py --workload c3_sbm1m --chunks 32 --reps 2 --tag c3 >> $o 2>&1
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv,noheader >> $o
cut -c1-160 $o
