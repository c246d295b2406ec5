# final round-1 capture of the dominant kernel on configs[3]: launch list of one timed filter
# pass and ncu --set full of one steady-state step launch (after the plain run exited 0)
CMD="python tools/sweep_filter.py --workload c3_sbm1m --chunks 32 --reps 1"
$CMD > gpurun_out/final_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 1000 --csv --log-file gpurun_out/final_launches.csv $CMD > gpurun_out/final_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:cheb_step -s 600 -c 1 -o gpurun_out/final_full $CMD > gpurun_out/final_full.log 2>&1
tail -n 3 gpurun_out/final_plain.log
