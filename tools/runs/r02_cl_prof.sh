# round 2: Chung-Lu step kernels under ncu --set full (one launch each, steady state), plus timings
o=gpurun_out/r02_chunglu_t.txt; : > $o
python tools/sweep_filter.py --workload x_chunglu1m --chunks 32 --reps 3 --tag base >> $o 2>&1
python tools/sweep_filter.py --workload c3_sbm1m --chunks 32 --reps 3 --tag c3 >> $o 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"hub_chunk_kernel|cheb_sell_kernel" -s 40 -c 2 -o gpurun_out/r02_chunglu_full \
  python tools/sweep_filter.py --workload x_chunglu1m --chunks 32 --reps 1 > /dev/null 2>&1; echo "ncu rc=$?"
