"""Debug helper: sc_cluster on configs[0] vs the oracle pipeline pieces."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1509_08863_b200 as sc
import scinputs
from oracle import ari as oari, laplacian, lambda_max, eigencount, chebyshev, kmeans

g = scinputs.sbm(2000, 5, 10, 0.1, seed=1234)
G = sc.Graph.from_csr(g)
lab = np.zeros(g.n, dtype=np.int32)
info = sc.sc_cluster(G.handle, 5, 32, 50, True, 32, 2024, 10, 100, False, lab)
print("info", info, "ari", oari.ari(lab, g.labels), "bincount", np.bincount(lab))
L = laplacian.laplacian(g)
ev = np.linalg.eigvalsh(L.toarray())
print("exact eig 1..8", ev[:8], "max", ev[-1])
lmax = info[0]
lk = info[1]
X = scinputs.gaussian_block(2024, g.n, 32)
Y = torch.empty((g.n, 32), dtype=torch.float32, device="cuda")
sc.sc_filter_lowpass_f32(G.handle, lk, lmax, 50, True, 32, 2024, None, Y)
Yg = Y.cpu().numpy()
Yo = chebyshev.lowpass_filter(L, X.astype(np.float64), lk, lmax, 50, True)
print("seeded filter rel err", np.linalg.norm(Yg - Yo) / np.linalg.norm(Yo), "norms", np.linalg.norm(Yg), np.linalg.norm(Yo))
u = np.stack([scinputs.uniforms(2024, 5, offset=5 * r) for r in range(10)])
lo, _, io, ito, ro, _ = kmeans.kmeans(Yo.astype(np.float32), 5, u, 100)
print("oracle kmeans ari", oari.ari(lo, g.labels), "inertia", io)
Fd = torch.from_numpy(Yo.astype(np.float32)).cuda()
lab2 = torch.empty(g.n, dtype=torch.int32, device="cuda")
print("gpu kmeans on oracle feats", sc.sc_kmeans(Fd, g.n, 32, 5, 10, 100, 2024, None, lab2), oari.ari(lab2.cpu().numpy(), g.labels))
mu = sc.sc_cheb_moments(G.handle, lmax, 50, 32, 2024 ^ 0x5e5e5e5e)
for c in [0.5, 1, 2, 3, 4, 6]:
    print("count", c, sc.sc_eigencount_from_moments(mu, 50, c, lmax, True), (ev <= c).sum())
