#!/bin/bash
# session 5: T_{s-1} block bulk-copied per tile (SC_SELL_BULKP=1) vs per-lane cp.async (default)
# (measured slower and reverted: apply the patch in profiles/r02_bulkp_rejected.md to rerun)
mkdir -p gpurun_out
o=gpurun_out/s5_bulkp.txt; : > $o
SC_SELL_BULKP=1 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "filter_f32_parity or filter_f64_parity or column_chunking or random_cases or moments_counts or full_size_c3" > gpurun_out/s5_bulkp_tests.log 2>&1
echo "parity (SC_SELL_BULKP=1): $(tail -n 1 gpurun_out/s5_bulkp_tests.log)" >> $o
for rep in 1 2; do
for v in 0 1; do
  echo "== SC_SELL_BULKP=$v" >> $o
  SC_SELL_BULKP=$v timeout 300 python tools/sweep_filter.py --workload c3_sbm1m --chunks 32 --reps 3 --tag bulkp$v 2>&1 | tail -n 2 | cut -c1-300 >> $o
done
done
for v in 0 1; do
  echo "== SC_SELL_BULKP=$v SC_SELL_FORCE_STAGES=3" >> $o
  SC_SELL_FORCE_STAGES=3 SC_SELL_SMEM_TARGET_KB=113 SC_SELL_BULKP=$v timeout 300 python tools/sweep_filter.py --workload c3_sbm1m --chunks 32 --reps 3 --tag bulkp${v}s3 2>&1 | tail -n 2 | cut -c1-300 >> $o
done
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw --format=csv >> $o
cat $o
