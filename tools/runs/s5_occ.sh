#!/bin/bash
# session 5: more consumer threads per SM (3-4 CTAs) at the price of register spills, small
# shared-memory plans; libs: native_build.py --defs "-DSC_SELL_MIN_CTAS=3|4 [-DSC_SELL_NC=12]"
mkdir -p gpurun_out
o=gpurun_out/s5_occ.txt; : > $o
run() { # lib stages dense
  SC_B200_LIB=paper_1509_08863_b200/$1 SC_SELL_FORCE_STAGES=$2 SC_SELL_FORCE_DENSE=$3 timeout 300 python tools/sweep_filter.py --workload c3_sbm1m --chunks 32 --reps 3 --tag "$1 st$2 dense$3" 2>&1 | tail -n 1 | cut -c1-170 >> $o
}
run libsc_b200.so 3 1
for lib in libsc_b200_m3nc12.so libsc_b200_m3.so libsc_b200_m4nc12.so; do
  run $lib 2 1; run $lib 2 0
done
run libsc_b200.so 2 0
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw --format=csv,noheader >> $o
cat $o
