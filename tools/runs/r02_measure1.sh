# round 2: bench line (configs[3]), gather-under-load probe, ncu of the SELL kernel (steady state),
# Chung-Lu launch list
o=gpurun_out/r02_measure1.txt; : > $o
python bench.py > gpurun_out/r02_bench_c3.json 2> gpurun_out/r02_bench_c3.err; echo "bench rc=$?" >> $o
./tools/gpl > gpurun_out/r02_gather_probe_load.txt 2>&1; echo "probe rc=$?" >> $o
python tools/sweep_filter.py --workload c3_sbm1m --chunks 32 --reps 1 --tag plain > gpurun_out/plain_c3.log 2>&1 && \
timeout 900 ncu --set full --cache-control none --clock-control none --import-source on -k regex:cheb_sell -s 600 -c 2 \
   -o gpurun_out/r02_sell_c3 python tools/sweep_filter.py --workload c3_sbm1m --chunks 32 --reps 1 --tag ncu > gpurun_out/ncu_c3.log 2>&1
echo "ncu full rc=$?" >> $o
python bench.py --no-e2e --no-cluster --no-stability --no-cpu-baseline --steps 2 --warmup 3 > gpurun_out/plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 1000 --csv --log-file gpurun_out/r02_c3_launches.csv \
   python bench.py --no-e2e --no-cluster --no-stability --no-cpu-baseline --steps 2 --warmup 3 > gpurun_out/ncu_launch.log 2>&1
echo "ncu launches rc=$?" >> $o
python tools/sweep_filter.py --workload x_chunglu1m --chunks 32 --reps 1 --tag plain > gpurun_out/cl_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"hub|sell" -s 400 -c 40 --csv \
  --log-file gpurun_out/r02_chunglu_launches.csv python tools/sweep_filter.py --workload x_chunglu1m --chunks 32 --reps 1 --tag ncu > gpurun_out/cl_ncu.log 2>&1
echo "ncu cl rc=$?" >> $o
