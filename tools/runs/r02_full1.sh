# round 2: full GPU test suite, Chung-Lu timing (split rows vs CSR kernel), bench.py default line
o=gpurun_out/r02_full1.txt; : > $o
nproc >> $o
( time timeout 2400 python -m pytest tests -m gpu -x -q --durations=15 ) >> $o 2>&1
echo "pytest rc=$?" >> $o
python tools/sweep_filter.py --workload x_chunglu1m --chunks 32 --reps 3 --tag sell >> $o 2>&1
SC_SELL=0 python tools/sweep_filter.py --workload x_chunglu1m --chunks 32 --reps 3 --tag csr >> $o 2>&1
python tools/sweep_filter.py --workload c3_sbm1m --chunks 32 --reps 3 --tag sell >> $o 2>&1
python bench.py > gpurun_out/r02_bench_c3.json 2> gpurun_out/r02_bench_c3.err; echo "bench rc=$?" >> $o
