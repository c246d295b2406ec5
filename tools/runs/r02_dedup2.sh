# round 2: ncu of the SELL kernel on the locality-rich graph, plain vs deduplicated gathers (64-column chunks)
SC_SELL_DEDUP=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"cheb_sell_kernel" -s 30 -c 1 -o gpurun_out/r02_rcm_plain \
  python tools/sweep_filter.py --workload x_gmm2d1m_rcm --chunks 64 --reps 1 > /dev/null 2>&1; echo "ncu rc=$?"
SC_SELL_DEDUP=2 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"cheb_sell_kernel" -s 30 -c 1 -o gpurun_out/r02_rcm_dedup \
  python tools/sweep_filter.py --workload x_gmm2d1m_rcm --chunks 64 --reps 1 > /dev/null 2>&1; echo "ncu rc=$?"
