#!/bin/bash
# gathers in flight (NB) x consumer warps (NC) x CTAs per SM, without register spills (the NB=2,
# NC=16 build spilled 208 B: the reason it measured slower); configs[3], 32-column chunks
o=gpurun_out/r02_nbnc.txt; : > $o
smi() { nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv,noheader >> $o; }
smi
for lib in libsc_b200.so libsc_b200_nb2nc12.so libsc_b200_nb3nc8.so libsc_b200_nb2nc8m3.so libsc_b200_nb2nc8.so libsc_b200.so; do
  SC_B200_LIB=paper_1509_08863_b200/$lib timeout 300 python tools/sweep_filter.py --workload c3_sbm1m --chunks 32 --reps 3 --tag $lib >> $o 2>&1
  smi
done
for lib in libsc_b200.so libsc_b200_nb2nc12.so libsc_b200_nb3nc8.so; do
  SC_B200_LIB=paper_1509_08863_b200/$lib timeout 300 python tools/sweep_filter.py --workload x_chunglu1m --chunks 32 --reps 2 --tag cl_$lib >> $o 2>&1
done
smi
cut -c1-200 $o
