#!/bin/bash
mkdir -p gpurun_out
o=gpurun_out/p2p_sell.log
timeout 1200 python -m pytest tests -m gpu -x -q -k "p2p or dist or partition or grid or emulated or rank or nccl" > $o 2>&1; echo "rc=$?" >> $o
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" >> $o 2>&1; echo "smoke_rc=$?" >> $o
timeout 900 python tools/grid_emulate.py c3_sbm1m 2,4,8 >> gpurun_out/p2p_sell_grid_c3.txt 2>&1
tail -12 $o; cat gpurun_out/p2p_sell_grid_c3.txt | cut -c1-300
