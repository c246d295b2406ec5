# round 2: deduplicated gathers -- parity, then timings on the locality-rich graph and configs[3]
python -m pytest tests -q -m gpu -x -k "filter and (dedup or streaming)" 2>&1 | tail -3
o=gpurun_out/r02_dedup1.txt; : > $o
for ch in 32 64; do
  python tools/sweep_filter.py --workload x_gmm2d1m_rcm --chunks $ch --reps 3 --tag dedup_auto >> $o 2>&1
  SC_SELL_DEDUP=0 python tools/sweep_filter.py --workload x_gmm2d1m_rcm --chunks $ch --reps 3 --tag plain >> $o 2>&1
done
python tools/sweep_filter.py --workload c3_sbm1m --chunks 32 --reps 3 --tag c3_auto >> $o 2>&1
SC_SELL_DEDUP=2 python tools/sweep_filter.py --workload c3_sbm1m --chunks 32 --reps 3 --tag c3_forced >> $o 2>&1
cat $o
