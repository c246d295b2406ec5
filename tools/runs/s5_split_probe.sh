#!/bin/bash
# session 5: role-split step probe (tools/split_role_probe.cu) on configs[3]'s CSR, beside the
# fused kernel's pass time on the same box
mkdir -p gpurun_out
o=gpurun_out/s5_split_probe.txt; : > $o
python -c "
import numpy as np
from scinputs import configs
g = configs.build_graph('c3_sbm1m')
np.asarray(g.row_ptr).astype(np.int64).tofile('/tmp/c3_rp.bin')
np.asarray(g.col_idx).astype(np.int32).tofile('/tmp/c3_ci.bin')
print(g.n, g.nnz)
"
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw --format=csv,noheader >> $o
timeout 300 ./tools/split_role_probe.bin /tmp/c3_rp.bin /tmp/c3_ci.bin 1000000 >> $o 2>&1; echo "rc=$?" >> $o
timeout 300 python tools/sweep_filter.py --workload c3_sbm1m --chunks 32 --reps 3 --tag fused_kernel 2>&1 | tail -n 1 | cut -c1-200 >> $o
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw --format=csv,noheader >> $o
rm -f /tmp/c3_rp.bin /tmp/c3_ci.bin
cat $o
