import os, sys
sys.path.insert(0, "/root/repo")
import torch, numpy as np
import paper_1509_08863_b200 as sc
from scinputs import configs
w = configs.WORKLOADS["c2_sbm100k"]
g = configs.build_graph("c2_sbm100k", cache=True)
G = sc.Graph.from_csr(g)
lmax = sc.sc_lambda_max(G.handle, 60, 0.01, 1)
lk, _ = sc.sc_estimate_lambda_k(G.handle, 20, lmax, w.order, True, 32, 2, 40, 1e-4)
Y = torch.empty((g.n, w.R), device="cuda")
sc.sc_filter_lowpass_f32(G.handle, lk, lmax, w.order, True, w.R, 3, None, Y)
lab = torch.empty(g.n, dtype=torch.int32, device="cuda")
res = sc.sc_kmeans(Y, g.n, w.R, 20, 5, 100, 4, None, lab)
print("iters", res[1])
