# round 2: Chung-Lu after the hub-partials change; c3 unchanged check; parity of split rows
python -m pytest tests -q -m gpu -x -k "filter and (split or chung or star)" 2>&1 | tail -2
o=gpurun_out/r02_chunglu_t2.txt; : > $o
python tools/sweep_filter.py --workload x_chunglu1m --chunks 32 --reps 3 --tag cl >> $o 2>&1
python tools/sweep_filter.py --workload c3_sbm1m --chunks 32 --reps 3 --tag c3 >> $o 2>&1
python tools/sweep_filter.py --workload x_chunglu1m --chunks 32 --reps 3 --tag cl >> $o 2>&1
cat $o
