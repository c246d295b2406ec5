#!/bin/bash
o=gpurun_out/r02_tune2.txt; : > $o
timeout 900 python -m pytest tests -m gpu -x -q -k "chunk_width or filter_f32 or filter_random or full_size_c3 or chunking" 2>&1 | tail -3 >> $o
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv,noheader >> $o
for wl in c3_sbm1m x_chunglu1m x_gmm2d1m_rcm x_sbm1m_eps005; do
  timeout 600 python tools/sweep_filter.py --workload $wl --chunks 0 --reps 3 --tag auto_$wl >> $o 2>&1
done
SC_CHUNK_WIDE=1 timeout 600 python tools/sweep_filter.py --workload x_sbm1m_eps005 --chunks 0 --reps 3 --tag wide_eps005 >> $o 2>&1
SC_CHUNK_WIDE=0 timeout 600 python tools/sweep_filter.py --workload x_sbm1m_eps005 --chunks 0 --reps 3 --tag narrow_eps005 >> $o 2>&1
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv,noheader >> $o
cut -c1-200 $o
