#!/bin/bash
# (1) configs[4] SELL launches under ncu: DRAM bytes per launch vs gathered bytes
# (2) the CSR step kernel's gathers in flight (EB) in the configs[4] 8-rank grid ranks
mkdir -p gpurun_out
o=gpurun_out/r02_c4_eb.txt; : > $o
smi() { nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv,noheader >> $o; }
smi
for lib in libsc_b200.so libsc_b200_eb4.so libsc_b200_eb3.so; do
  SC_B200_LIB=paper_1509_08863_b200/$lib timeout 900 python tools/grid_emulate.py c4_sbm10m 8 2>&1 | grep '"grid"' | sed "s/^/$lib /" >> $o
  smi
done
python tools/sweep_filter.py --workload c4_sbm10m --chunks 0 --reps 1 --tag c4 > gpurun_out/c4d_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second \
    --clock-control none -k regex:cheb_sell -s 40 -c 4 --csv --log-file gpurun_out/c4d_ncu.csv \
    python tools/sweep_filter.py --workload c4_sbm10m --chunks 0 --reps 1 --tag c4 > gpurun_out/c4d_ncu.log 2>&1
echo "ncu_rc=$?" >> $o
tail -2 gpurun_out/c4d_plain.log >> $o
cut -c1-300 $o
