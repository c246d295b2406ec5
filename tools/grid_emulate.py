"""Per-rank compute of the multi-GPU decompositions, emulated on one GPU (GPU box).

    python tools/grid_emulate.py [workload] [worlds, e.g. 2,4,8]

For every world size and both decompositions -- pure row partition (1 column group) and the
2-D grid bench.py picks (dist.grid_shape) -- one column group's n_row ranks run the fused
peer-store filter on this GPU (sc_p2p_filter_group_f32: the ranks' step kernels one after
another, peer stores into local memory), so time / n_row is a rank's compute time with the
exchange free.  Printed beside it: the halo rows a rank receives per pass (the NVLink traffic
the exchange adds) and their time at 900 GB/s per direction (NVLink 5 nominal).  One JSON
line per configuration."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1509_08863_b200 as sc
from paper_1509_08863_b200 import dist as pdist
from scinputs import configs

wl = sys.argv[1] if len(sys.argv) > 1 else "c3_sbm1m"
worlds = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "2,4,8").split(",")]
w = configs.WORKLOADS[wl]
g = configs.build_graph(wl, cache=True)
n, R, order = g.n, w.R, w.order
lmax = 2.0 * float(g.degrees().max())
d = sc.sc_cheby_coeffs(0.05 * lmax, lmax, order, w.jackson)
# optional third argument: the column-group counts to try (e.g. 1,2,4,8); default: the pure row
# partition and the grid bench.py picks (dist.grid_shape)
cg_list = [int(x) for x in sys.argv[3].split(",")] if len(sys.argv) > 3 else None
for world in worlds:
    variants = ((("rows", 1), ("grid", None)) if cg_list is None else
                tuple((f"grid{c}", c) for c in cg_list if world % c == 0 and R % c == 0 and (R // c) % 4 == 0))
    for label, cgs in variants:
        n_cg, n_row = pdist.grid_shape(world, R, col_groups=cgs)
        if label == "grid" and n_cg == 1:
            continue
        c0, c1 = pdist.column_range(R, n_cg, 0)
        t0 = time.perf_counter()
        grp = pdist.P2PGroup(g.row_ptr, g.col_idx, g.values, n, n_row, c1 - c0)
        setup = time.perf_counter() - t0
        Xs = [torch.randn((p.n_local, c1 - c0), device="cuda") for p in grp.parts]
        Ys = [torch.empty_like(x) for x in Xs]
        grp.filter(d, order, lmax, Xs, Ys)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(2):
            grp.filter(d, order, lmax, Xs, Ys)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 2
        halo = max(p.n_halo for p in grp.parts)
        halo_bytes = halo * (c1 - c0) * 4 * order
        nv_ms = halo_bytes / 900e9 * 1e3
        print(json.dumps({"workload": wl, "world": world, "decomposition": label, "col_groups": n_cg,
                          "row_blocks": n_row, "cols_per_rank": c1 - c0,
                          "rank_compute_ms_per_pass": round(ms / n_row, 3),
                          "max_halo_rows": int(halo), "halo_GB_per_pass": round(halo_bytes / 1e9, 3),
                          "halo_ms_at_900GBps": round(nv_ms, 3),
                          "predicted_ms_per_pass": round(max(ms / n_row, nv_ms), 3), "setup_s": round(setup, 1)}),
              flush=True)
        grp.close()
        del Xs, Ys
        torch.cuda.empty_cache()
