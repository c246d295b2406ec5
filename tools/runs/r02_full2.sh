# round 2: full GPU suite; Chung-Lu split-row thresholds
o=gpurun_out/r02_full2.txt; : > $o
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv >> $o
for h in 512 256 128 64; do
  SC_SELL_HUB_DEG=$h python tools/sweep_filter.py --workload x_chunglu1m --chunks 32 --reps 3 --tag hub$h >> $o 2>&1
done
python tools/sweep_filter.py --workload c3_sbm1m --chunks 32 --reps 3 --tag c3 >> $o 2>&1
( time timeout 2400 python -m pytest tests -m gpu -x -q --durations=15 ) >> $o 2>&1
echo "pytest rc=$?" >> $o
