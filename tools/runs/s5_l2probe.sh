#!/bin/bash
# session 5: L2 -> SM throughput probe, incl. configs[3]'s own column-index stream (pure gathers)
mkdir -p gpurun_out
python -c "
import numpy as np
from scinputs import configs
g = configs.build_graph('c3_sbm1m')
np.asarray(g.col_idx).astype(np.int32).tofile('/tmp/c3_idx.bin')
print(g.n, g.nnz)
"
timeout 500 ./tools/l2_cap_probe.bin /tmp/c3_idx.bin 1000000 > gpurun_out/l2_cap_probe.txt 2>&1; echo rc=$?
rm -f /tmp/c3_idx.bin
cat gpurun_out/l2_cap_probe.txt
