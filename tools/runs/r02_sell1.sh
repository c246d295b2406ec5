# round 2: first SELL-kernel run: filter parity + c3 timing vs the CSR kernel and variants
L=paper_1509_08863_b200
o=gpurun_out/r02_sell1.txt; : > $o
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "filter or full_size_c3 or cheb_step or random_cases" >> $o 2>&1
echo "pytest rc=$?" >> $o
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv >> $o
python tools/sweep_filter.py --workload c3_sbm1m --chunks 16,32,64 --reps 3 --tag sell >> $o 2>&1
SC_SELL=0 python tools/sweep_filter.py --workload c3_sbm1m --chunks 32 --reps 3 --tag csr >> $o 2>&1
SC_B200_LIB=$PWD/$L/libsc_b200_nc12.so python tools/sweep_filter.py --workload c3_sbm1m --chunks 16,32,64 --reps 3 --tag sell_nc12 >> $o 2>&1
SC_B200_LIB=$PWD/$L/libsc_b200_nb1.so python tools/sweep_filter.py --workload c3_sbm1m --chunks 16,32 --reps 3 --tag sell_nb1 >> $o 2>&1
python tools/sweep_filter.py --workload c3_sbm1m --chunks 16,32 --reps 3 --dtype f64 --tag sell_f64 >> $o 2>&1
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv >> $o
