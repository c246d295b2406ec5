#!/bin/bash
mkdir -p gpurun_out
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv > gpurun_out/grid_c4_sell.txt
timeout 2400 python tools/grid_emulate.py c4_sbm10m 2,4,8 >> gpurun_out/grid_c4_sell.txt 2>&1
SC_SELL=0 timeout 1200 python tools/grid_emulate.py c4_sbm10m 8 | sed 's/^/csr /' >> gpurun_out/grid_c4_sell.txt 2>&1
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv >> gpurun_out/grid_c4_sell.txt
cut -c1-300 gpurun_out/grid_c4_sell.txt
