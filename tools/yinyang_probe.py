"""Would per-group (Yinyang) bounds skip work on configs[3] features?  (GPU box, torch fp64
Lloyd on the sc_cluster features; counts how many (point, centroid-group) pairs a Yinyang
filter would have to rescan per iteration, groups = G blocks of consecutive centroids after
sorting the initial centroids along their first principal direction.)"""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1509_08863_b200 as sc
from scinputs import configs

w = configs.WORKLOADS["c3_sbm1m"]
g = configs.build_graph("c3_sbm1m", cache=True)
G = sc.Graph.from_csr(g)
lmax = sc.sc_lambda_max(G.handle, 60, 0.01, 1)
lk, _ = sc.sc_estimate_lambda_k(G.handle, w.k, lmax, w.order, True, 32, 2, 40, 1e-4)
Y = torch.empty((g.n, w.R), dtype=torch.float32, device="cuda")
sc.sc_filter_lowpass_f32(G.handle, lk, lmax, w.order, w.jackson, w.R, 3, None, Y)
X = Y.double()
k = w.k
torch.manual_seed(0)
C = X[torch.randperm(g.n, device="cuda")[:k]].clone()
out = {}
for ng in (13, 25):
    Cg = C.clone()
    # groups: sort centroids by projection on the top principal direction, ng contiguous blocks
    u, s_, v = torch.pca_lowrank(Cg, q=1)
    order = torch.argsort(Cg @ v[:, 0])
    grp = torch.empty(k, dtype=torch.long, device="cuda")
    grp[order] = torch.arange(k, device="cuda") * ng // k
    D = torch.cdist(X, Cg)
    lab = D.argmin(1)
    ub = D.gather(1, lab[:, None])[:, 0]
    lb = torch.full((g.n, ng), float("inf"), dtype=torch.float64, device="cuda")
    for gi in range(ng):
        m = (grp == gi)
        Dg = D[:, m].clone()
        own = (grp[lab] == gi)
        idx = torch.nonzero(m)[:, 0]
        Dg[own, (idx[None, :] == lab[own, None]).float().argmax(1)] = float("inf")
        lb[:, gi] = Dg.min(1).values
    rescans = []
    for it in range(30):
        newC = torch.zeros_like(Cg).index_add_(0, lab, X)
        cnt = torch.bincount(lab, minlength=k).clamp(min=1)[:, None].double()
        newC = newC / cnt
        shift = (newC - Cg).norm(dim=1)
        Cg = newC
        gshift = torch.zeros(ng, dtype=torch.float64, device="cuda").scatter_reduce(0, grp, shift, "amax")
        lb = lb - gshift[None, :]
        D = torch.cdist(X, Cg)
        dlab = D.gather(1, lab[:, None])[:, 0]
        fail = lb < dlab[:, None]               # groups a Yinyang filter must rescan
        rescans.append(round(float(fail.float().mean()), 4))
        lab = D.argmin(1)
        for gi in range(ng):                      # refresh bounds (exact, for the probe)
            m = (grp == gi)
            Dg = D[:, m].clone()
            own = (grp[lab] == gi)
            idx = torch.nonzero(m)[:, 0]
            Dg[own, (idx[None, :] == lab[own, None]).float().argmax(1)] = float("inf")
            lb[:, gi] = torch.minimum(lb[:, gi], Dg.min(1).values) if False else Dg.min(1).values
    out[f"groups_{ng}"] = rescans
print(json.dumps(out))
