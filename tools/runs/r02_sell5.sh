# round 2: SELL with per-plan stages / dense staging (runtime), parity + configs[3] timing
o=gpurun_out/r02_sell5.txt; : > $o
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "filter or full_size_c3 or cheb_step or random_cases or cluster or partitioned" >> $o 2>&1
echo "pytest rc=$?" >> $o
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv >> $o
python tools/sweep_filter.py --workload c3_sbm1m --chunks 16,32 --reps 3 --tag auto >> $o 2>&1
for cfg in "3 1" "2 1" "3 0" "2 0"; do set -- $cfg
  SC_SELL_FORCE_STAGES=$1 SC_SELL_FORCE_DENSE=$2 python tools/sweep_filter.py --workload c3_sbm1m --chunks 16,32 --reps 3 --tag st$1_dense$2 >> $o 2>&1
  SC_SELL_FORCE_STAGES=$1 SC_SELL_FORCE_DENSE=$2 python tools/time_weighted.py 2>&1 | sed "s/^/st$1_dense$2 /" >> $o
done
python tools/time_weighted.py 2>&1 | sed "s/^/auto /" >> $o
python tools/sweep_filter.py --workload c3_sbm1m --chunks 16 --reps 2 --dtype f64 --tag auto_f64 >> $o 2>&1
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv >> $o
