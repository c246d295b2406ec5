#!/bin/bash
# round 2 (session 3): gathers in flight (NB) against the shared memory left to L1, configs[3]
o=gpurun_out/r02_nb_smem.txt; : > $o
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv >> $o
for lib in libsc_b200.so libsc_b200_nb2.so libsc_b200_nb3.so; do
  for cfg in "3 1" "2 1" "2 0"; do set -- $cfg
    SC_B200_LIB=paper_1509_08863_b200/$lib SC_SELL_FORCE_STAGES=$1 SC_SELL_FORCE_DENSE=$2 timeout 300 \
      python tools/sweep_filter.py --workload c3_sbm1m --chunks 32 --reps 3 --tag ${lib}_st$1_dense$2 >> $o 2>&1
  done
done
SC_B200_LIB=paper_1509_08863_b200/libsc_b200.so timeout 300 python tools/sweep_filter.py --workload c3_sbm1m --chunks 32 --reps 3 --tag again_default >> $o 2>&1
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv >> $o
cat $o | cut -c1-400
