# round 2: SELL defaults (NB 1, plan-sized stages): parity subset, configs[3] f32/f64, weighted
# pattern, locality-rich graphs (2-D GMM kNN in RCM order, SBM eps 0.005)
o=gpurun_out/r02_sell3.txt; : > $o
nproc >> $o
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "filter or full_size_c3 or cheb_step or random_cases or cluster" >> $o 2>&1
echo "pytest rc=$?" >> $o
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv >> $o
python tools/sweep_filter.py --workload c3_sbm1m --chunks 16,32 --reps 3 --tag sell >> $o 2>&1
python tools/sweep_filter.py --workload c3_sbm1m --chunks 16 --reps 2 --dtype f64 --tag sell_f64 >> $o 2>&1
python tools/time_weighted.py >> $o 2>&1
SC_SELL=0 python tools/time_weighted.py >> $o 2>&1
python tools/sweep_filter.py --workload x_gmm2d1m_rcm --chunks 32,64 --reps 3 --tag sell >> $o 2>&1
SC_SELL=0 python tools/sweep_filter.py --workload x_gmm2d1m_rcm --chunks 32,64 --reps 3 --tag csr >> $o 2>&1
python tools/sweep_filter.py --workload x_sbm1m_eps005 --chunks 32,64 --reps 3 --tag sell >> $o 2>&1
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv >> $o
