# round 2: 24-column chunks (96 MB gathered table, fits L2) vs 32 on configs[3]
o=gpurun_out/r02_ch24.txt; : > $o
for r in 1 2; do python tools/sweep_filter.py --workload c3_sbm1m --chunks 32,24,48,16 --reps 3 --tag r$r >> $o 2>&1; done
cat $o
