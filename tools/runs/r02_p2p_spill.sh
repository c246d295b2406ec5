#!/bin/bash
# SELL fused-exchange epilogue without spills (Y stored before the peer stores): per-rank compute
o=gpurun_out/r02_p2p_spill.txt; : > $o
timeout 900 python -m pytest tests -m gpu -x -q -k "p2p or partition or grid or emulated" 2>&1 | tail -2 >> $o
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv,noheader >> $o
timeout 900 python tools/grid_emulate.py c3_sbm1m 4,8 >> $o 2>&1
SC_SELL=0 timeout 900 python tools/grid_emulate.py c3_sbm1m 8 2>&1 | sed 's/^/csr /' >> $o
timeout 1500 python tools/grid_emulate.py c4_sbm10m 8 2>&1 | grep '"grid"' >> $o
SC_P2P_SELL_WIDE=1 timeout 1500 python tools/grid_emulate.py c4_sbm10m 8 2>&1 | grep '"grid"' | sed 's/^/sellwide /' >> $o
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv,noheader >> $o
cut -c1-330 $o
