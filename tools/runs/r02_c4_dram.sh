#!/bin/bash
# configs[4] SELL launches: DRAM bytes per launch vs the gathered bytes (is the kernel at the
# HBM roofline of the traffic a random-gather SpMM must move?)
mkdir -p gpurun_out
python tools/sweep_filter.py --workload c4_sbm10m --chunks 0 --reps 1 --tag c4 > gpurun_out/c4d_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second \
    --clock-control none -k regex:cheb_sell -s 40 -c 4 --csv --log-file gpurun_out/c4d_ncu.csv \
    python tools/sweep_filter.py --workload c4_sbm10m --chunks 0 --reps 1 --tag c4 > gpurun_out/c4d_ncu.log 2>&1
echo "rc=$?"; cat gpurun_out/c4d_plain.log | tail -2; grep -v '^==' gpurun_out/c4d_ncu.csv | cut -d, -f5,13-15 | head -40
