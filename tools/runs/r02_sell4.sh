# round 2: shared-memory footprint variants of the SELL kernel (L1 = 228 KB - shared memory
# holds the gathers in flight): dense staging off (d0), 2 stages (s2), 12 consumer warps
L=paper_1509_08863_b200
o=gpurun_out/r02_sell4.txt; : > $o
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv >> $o
for v in default d0 s2 d0s2 d0nc12 nc12 d0s2nb2; do
  lib=$PWD/$L/libsc_b200_$v.so; [ $v = default ] && lib=$PWD/$L/libsc_b200.so
  SC_B200_LIB=$lib python tools/sweep_filter.py --workload c3_sbm1m --chunks 16,32 --reps 3 --tag $v >> $o 2>&1
  SC_B200_LIB=$lib python tools/time_weighted.py 2>&1 | sed "s/^/$v /" >> $o
  SC_B200_LIB=$lib python tools/sweep_filter.py --workload x_gmm2d1m_rcm --chunks 64 --reps 3 --tag $v >> $o 2>&1
done
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv >> $o
