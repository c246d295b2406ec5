# round 2: full GPU suite; Chung-Lu launch list (hub vs SELL kernel share)
o=gpurun_out/r02_full3.txt; : > $o
( time timeout 2400 python -m pytest tests -m gpu -x -q --durations=20 ) >> $o 2>&1
echo "pytest rc=$?" >> $o
SC_SELL_HUB_DEG=128 python tools/sweep_filter.py --workload x_chunglu1m --chunks 32 --reps 1 --tag hub128 > gpurun_out/cl_plain.log 2>&1 && \
SC_SELL_HUB_DEG=128 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"hub|sell" -s 400 -c 40 --csv \
  --log-file gpurun_out/r02_chunglu_launches.csv python tools/sweep_filter.py --workload x_chunglu1m --chunks 32 --reps 1 --tag ncu > gpurun_out/cl_ncu.log 2>&1
echo "ncu rc=$?" >> $o
