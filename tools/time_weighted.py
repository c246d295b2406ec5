"""Weighted-graph filter timing (GPU box): configs[3]'s SBM pattern with symmetric random
weights in (0, 1] (the streaming kernel's weighted variant), one fp32 pass of p = 200 steps
over R = 64 columns, median of 3 after a warm-up pass."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import scipy.sparse as sp
import paper_1509_08863_b200 as sc
from scinputs import configs

g = configs.build_graph("c3_sbm1m", cache=True)
n = g.n
A = sp.csr_matrix((np.ones(g.nnz, np.float32), g.col_idx, g.row_ptr), shape=(n, n))
rng = np.random.default_rng(5)
U = sp.triu(A, 1).tocoo()
w = rng.uniform(0.05, 1.0, U.nnz).astype(np.float32)
Wm = sp.coo_matrix((w, (U.row, U.col)), shape=(n, n))
Wm = (Wm + Wm.T).tocsr()
Wm.sort_indices()
G = sc.Graph(n, Wm.indptr.astype(np.int64), Wm.indices.astype(np.int32), Wm.data.astype(np.float32))
lmax = 2.0 * G.info()[3]
R, order = 64, 200
d = sc.sc_cheby_coeffs(0.01 * lmax, lmax, order, False)
X = torch.randn((n, R), device="cuda")
Y = torch.empty_like(X)
sc.sc_filter_apply_f32(G.handle, d, order, lmax, R, X, Y)
ts = []
for _ in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    sc.sc_filter_apply_f32(G.handle, d, order, lmax, R, X, Y)
    e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
print(json.dumps({"graph": "c3 pattern, random symmetric weights", "nnz": int(Wm.nnz), "ms_per_pass": sorted(ts)[1]}))
