# round 2: hub kernel (16 gathers in flight), parity of the split-row paths, configs[3] launch list of a timed pass
o=gpurun_out/r02_measure2.txt; : > $o
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "filter or random_cases" >> $o 2>&1
echo "pytest rc=$?" >> $o
python tools/sweep_filter.py --workload x_chunglu1m --chunks 32 --reps 3 --tag cl >> $o 2>&1
python tools/sweep_filter.py --workload c3_sbm1m --chunks 32 --reps 3 --tag c3 >> $o 2>&1
python tools/sweep_filter.py --workload x_chunglu1m --chunks 32 --reps 1 --tag plain > gpurun_out/cl_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"hub|sell" -s 400 -c 40 --csv \
  --log-file gpurun_out/r02_chunglu_launches.csv python tools/sweep_filter.py --workload x_chunglu1m --chunks 32 --reps 1 --tag ncu > gpurun_out/cl_ncu.log 2>&1
echo "ncu cl rc=$?" >> $o
python tools/sweep_filter.py --workload c3_sbm1m --chunks 32 --reps 1 --tag plain > gpurun_out/c3_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 420 -c 420 --csv \
  --log-file gpurun_out/r02_c3_launches.csv python tools/sweep_filter.py --workload c3_sbm1m --chunks 32 --reps 1 --tag ncu > gpurun_out/c3_ncu.log 2>&1
echo "ncu c3 rc=$?" >> $o
