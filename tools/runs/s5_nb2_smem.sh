#!/bin/bash
# session 5: 8 gathers in flight per lane (NB = 2) with 12 / 14 consumer warps x 2 CTAs AND small
# shared-memory plans (more L1 for the loads in flight; r02_nbnc.sh ran them on the default plan)
# libs: native_build.py --defs "-DSC_SELL_NB=2 -DSC_SELL_NC=12|14" --out .../libsc_b200_nb2nc12|14.so
mkdir -p gpurun_out
o=gpurun_out/s5_nb2_smem.txt; : > $o
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw --format=csv,noheader >> $o
run() { # lib stages dense
  SC_B200_LIB=paper_1509_08863_b200/$1 SC_SELL_FORCE_STAGES=$2 SC_SELL_FORCE_DENSE=$3 timeout 300 python tools/sweep_filter.py --workload c3_sbm1m --chunks 32 --reps 3 --tag "$1 st$2 dense$3" 2>&1 | tail -n 1 | cut -c1-200 >> $o
}
run libsc_b200.so 3 1
for lib in libsc_b200_nb2nc12.so libsc_b200_nb2nc14.so; do
  run $lib 3 1; run $lib 2 1; run $lib 2 0
done
run libsc_b200.so 2 1
run libsc_b200.so 3 1
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw --format=csv,noheader >> $o
cat $o
