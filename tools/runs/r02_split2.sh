# round 2: split off by default; sigma / hub threshold on Chung-Lu; configs repeat for box comparison
o=gpurun_out/r02_split2.txt; : > $o
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv >> $o
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "pipeline or partitioned or dist_kmeans or halves" >> $o 2>&1
echo "pytest rc=$?" >> $o
python tools/sweep_filter.py --workload c3_sbm1m --chunks 16,32 --reps 3 --tag c3 >> $o 2>&1
python tools/sweep_filter.py --workload x_chunglu1m --chunks 32 --reps 3 --tag cl_sigma4096 >> $o 2>&1
SC_SELL_SIGMA=64 python tools/sweep_filter.py --workload x_chunglu1m --chunks 32 --reps 3 --tag cl_sigma64 >> $o 2>&1
SC_SELL_SIGMA=1024 python tools/sweep_filter.py --workload x_chunglu1m --chunks 32 --reps 3 --tag cl_sigma1024 >> $o 2>&1
SC_SELL_HUB_DEG=256 python tools/sweep_filter.py --workload x_chunglu1m --chunks 32 --reps 3 --tag cl_hub256 >> $o 2>&1
python tools/time_weighted.py 2>&1 | sed "s/^/weighted /" >> $o
python tools/sweep_filter.py --workload x_gmm2d1m_rcm --chunks 32,64 --reps 3 --tag knn >> $o 2>&1
python tools/sweep_filter.py --workload x_sbm1m_eps005 --chunks 32 --reps 3 --tag eps005 >> $o 2>&1
python tools/sweep_filter.py --workload c3_sbm1m --chunks 16 --reps 2 --dtype f64 --tag f64 >> $o 2>&1
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv >> $o
