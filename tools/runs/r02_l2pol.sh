# round 2: L2 eviction-policy sweep of the step kernel on configs[3] (c3_sbm1m)
# SC_L2POL = own + 4*next + 16*prev: own {0 first,1 normal,2 last}, next {0 none,1 first,2 last,3 normal}, prev {0 first,1 normal}
L=paper_1509_08863_b200
o=gpurun_out/r02_l2pol.txt; : > $o
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv >> $o
python tools/sweep_filter.py --workload c3_sbm1m --chunks 16,32 --pols 0,1,4,5,6,9,10 --reps 2 --tag default >> $o 2>&1
SC_B200_LIB=$PWD/$L/libsc_b200_gl.so python tools/sweep_filter.py --workload c3_sbm1m --chunks 16,32 --pols 0,4,5,6,10 --reps 2 --tag gatherlast >> $o 2>&1
SC_L2_SETASIDE_MB=79 SC_B200_LIB=$PWD/$L/libsc_b200_gl.so python tools/sweep_filter.py --workload c3_sbm1m --chunks 16,24,32 --pols 0,4,5,6,10 --reps 2 --tag gatherlast_setaside >> $o 2>&1
SC_L2_SETASIDE_MB=79 python tools/sweep_filter.py --workload c3_sbm1m --chunks 16,32 --pols 0,5,6,10 --reps 2 --tag setaside >> $o 2>&1
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv >> $o
