# round 2: configs[4] bench line with sc_cluster, grid emulation of the multi-GPU decompositions on
# configs[4], Chung-Lu split-row thresholds
o=gpurun_out/r02_c4.txt; : > $o
for h in 256 512; do SC_SELL_HUB_DEG=$h python tools/sweep_filter.py --workload x_chunglu1m --chunks 32 --reps 3 --tag hub$h >> $o 2>&1; done
python tools/sweep_filter.py --workload x_chunglu1m --chunks 32 --reps 3 --tag hub128 >> $o 2>&1
python bench.py --workload c4_sbm10m --steps 3 --warmup 3 --no-stability > gpurun_out/r02_bench_c4.json 2> gpurun_out/r02_bench_c4.err; echo "bench c4 rc=$?" >> $o
timeout 2400 python tools/grid_emulate.py c4_sbm10m 2,4,8 > gpurun_out/r02_grid_emulate_c4.txt 2>&1; echo "grid rc=$?" >> $o
