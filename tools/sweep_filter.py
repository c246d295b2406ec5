"""Timing sweep of the fused filter on one workload (GPU box).

    SC_B200_LIB=<lib.so> python tools/sweep_filter.py --workload c3_sbm1m \
        --chunks 16,32 --l2flags 0,1 [--reps 3]

Each configuration: p fused steps over the resident N x R block (one filter pass),
timed with CUDA events after one warm-up pass; prints one JSON line per config.
The graph is cached under $SC_GRAPH_CACHE (default /tmp/sc_graphs) between processes.
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import paper_1509_08863_b200 as sc
from scinputs import configs


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c3_sbm1m")
    ap.add_argument("--chunks", default="16,32")
    ap.add_argument("--l2flags", default="0", help="(removed experiment knob, ignored)")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--dtype", default="f32")
    ap.add_argument("--tag", default="")
    ap.add_argument("--pols", default="", help="comma list of SC_L2POL values to sweep (experiment knob)")
    a = ap.parse_args()
    w = configs.WORKLOADS[a.workload]
    g = configs.build_graph(a.workload, cache=True)
    G = sc.Graph.from_csr(g)
    n, R, order = g.n, w.R, w.order
    smax = G.info()[3]
    lmax = 2.0 * smax
    d = sc.sc_cheby_coeffs(0.01 * lmax, lmax, order, w.jackson)
    dt = torch.float32 if a.dtype == "f32" else torch.float64
    X = torch.randn((n, R), dtype=dt, device="cuda")
    Y = torch.empty_like(X)
    f = sc.sc_filter_apply_f32 if a.dtype == "f32" else sc.sc_filter_apply_f64
    nnz_l = g.nnz + n
    pols = a.pols.split(",") if a.pols else [os.environ.get("SC_L2POL", "0")]
    for ch in a.chunks.split(","):
        for fl in pols:
            os.environ["SC_CHUNK"] = ch
            os.environ["SC_L2POL"] = fl
            f(G.handle, d, order, lmax, R, X, Y)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            sc.sc_profile_begin()
            e0.record()
            for _ in range(a.reps):
                f(G.handle, d, order, lmax, R, X, Y)
            e1.record()
            torch.cuda.synchronize()
            launches, steps, kms, abytes = sc.sc_profile_end()
            ms = e0.elapsed_time(e1) / a.reps
            print(json.dumps({"tag": a.tag, "workload": a.workload, "dtype": a.dtype, "chunk": int(ch),
                              "l2pol": int(fl), "ms_per_pass": round(ms, 3),
                              "value": nnz_l * R * order / (ms / 1e3),
                              "algo_GBps": abytes / (kms / 1e3) / 1e9, "step_launches": steps // a.reps}),
                  flush=True)


if __name__ == "__main__":
    main()
