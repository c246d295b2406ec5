# round 2: split gather (column halves) + sigma windows + hub kernel with staged indices
o=gpurun_out/r02_split1.txt; : > $o
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv >> $o
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "filter or full_size_c3 or cheb_step or random_cases" >> $o 2>&1
echo "pytest rc=$?" >> $o
python tools/sweep_filter.py --workload c3_sbm1m --chunks 32 --reps 3 --tag split_auto >> $o 2>&1
SC_SELL_SPLIT=0 python tools/sweep_filter.py --workload c3_sbm1m --chunks 32 --reps 3 --tag nosplit >> $o 2>&1
SC_SELL_SPLIT=2 python tools/sweep_filter.py --workload c3_sbm1m --chunks 16,64 --reps 3 --tag split_forced >> $o 2>&1
python tools/sweep_filter.py --workload c3_sbm1m --chunks 16 --reps 3 --dtype f64 --tag f64_auto >> $o 2>&1
python tools/sweep_filter.py --workload x_chunglu1m --chunks 32 --reps 3 --tag cl_sigma >> $o 2>&1
SC_SELL_SIGMA=64 python tools/sweep_filter.py --workload x_chunglu1m --chunks 32 --reps 3 --tag cl_nosigma >> $o 2>&1
python tools/time_weighted.py 2>&1 | sed "s/^/weighted /" >> $o
python tools/sweep_filter.py --workload x_gmm2d1m_rcm --chunks 32,64 --reps 3 --tag knn >> $o 2>&1
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv >> $o
