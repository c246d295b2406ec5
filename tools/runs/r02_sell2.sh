# round 2: SELL kernel variants on configs[3] (timing) + steady-state ncu captures of two variants
L=paper_1509_08863_b200
o=gpurun_out/r02_sell2.txt; : > $o
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv >> $o
python tools/sweep_filter.py --workload c3_sbm1m --chunks 16,32 --reps 3 --tag nb2 >> $o 2>&1
for v in nb1 nb1nc12 nb1na nb1s64 nb2na nb1cg nb2s64; do
  SC_B200_LIB=$PWD/$L/libsc_b200_$v.so python tools/sweep_filter.py --workload c3_sbm1m --chunks 16,24,32 --reps 3 --tag $v >> $o 2>&1
done
SC_B200_LIB=$PWD/$L/libsc_b200_f64nb1.so python tools/sweep_filter.py --workload c3_sbm1m --chunks 16,32 --reps 2 --dtype f64 --tag f64nb1 >> $o 2>&1
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv >> $o
for v in nb1 nb2; do
  lib=$PWD/$L/libsc_b200_$v.so; [ $v = nb2 ] && lib=$PWD/$L/libsc_b200.so
  SC_B200_LIB=$lib python tools/sweep_filter.py --workload c3_sbm1m --chunks 32 --reps 1 --tag plain_$v > gpurun_out/plain_$v.log 2>&1 && \
  SC_B200_LIB=$lib timeout 600 ncu --set full --cache-control none --clock-control none --import-source on -k regex:cheb_sell -s 600 -c 2 \
     -o gpurun_out/r02_sell_$v python tools/sweep_filter.py --workload c3_sbm1m --chunks 32 --reps 1 --tag ncu_$v > gpurun_out/ncu_$v.log 2>&1
  echo "ncu $v rc=$?" >> $o
done
