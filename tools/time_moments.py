"""Moments pass vs a SELL fp64 filter pass of the same width (GPU box; tooling).

sc_cheb_moments (order p, n_probe probes, fp64, plain-CSR MOMENTS step kernel) against
sc_filter_apply_f64 on an N x n_probe block with the same order (SELL step kernel)."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1509_08863_b200 as sc
from scinputs import configs

wl = sys.argv[1] if len(sys.argv) > 1 else "c3_sbm1m"
P = int(sys.argv[2]) if len(sys.argv) > 2 else 32
w = configs.WORKLOADS[wl]
g = configs.build_graph(wl, cache=True)
G = sc.Graph.from_csr(g)
lmax = 2.0 * G.info()[3]
order = w.order
mu = np.zeros(2 * order + 1)
for rep in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    mu = sc.sc_cheb_moments(G.handle, lmax, order, P, 7)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    print(json.dumps({"what": "moments", "P": P, "order": order, "ms": round((t1 - t0) * 1e3, 2)}), flush=True)
d = sc.sc_cheby_coeffs(0.01 * lmax, lmax, order, False)
X = torch.randn((g.n, P), dtype=torch.float64, device="cuda")
Y = torch.empty_like(X)
for rep in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    sc.sc_filter_apply_f64(G.handle, d, order, lmax, P, X, Y)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    print(json.dumps({"what": "filter_f64", "P": P, "order": order, "ms": round((t1 - t0) * 1e3, 2)}), flush=True)
