"""k-means on configs[4]-shaped features (GPU box, tooling): the tensor screen with the wide
register prefetch (SC_KMEANS_TC_WIDE=1), with two tiles per CTA (SC_KMEANS_TC_PAIR=1), against the narrow
kernel's staging loads; labels,
centroids and inertia must be identical."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1509_08863_b200 as sc
from scinputs import configs

wl = sys.argv[1] if len(sys.argv) > 1 else "c4_sbm10m"
restarts = int(sys.argv[2]) if len(sys.argv) > 2 else 10
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 20
w = configs.WORKLOADS[wl]
t0 = time.perf_counter()
g = configs.build_graph(wl, cache=True)
print(f"graph {time.perf_counter() - t0:.1f} s", flush=True)
G = sc.Graph.from_csr(g)
n, R = g.n, w.R
lmax = 2.0 * G.info()[3]
Y = torch.empty((n, R), dtype=torch.float32, device="cuda")
sc.sc_filter_lowpass_f32(G.handle, 0.005 * lmax, lmax, w.order, w.jackson, R, 3, None, Y)
del G
out = {}
for wide, pair in (("1", "1"), ("1", "0"), ("0", "1"), ("1", "1")):
    os.environ["SC_KMEANS_TC_WIDE"] = wide
    os.environ["SC_KMEANS_TC_PAIR"] = pair
    lab = torch.empty(n, dtype=torch.int32, device="cuda")
    C = np.zeros((w.k, R), dtype=np.float64)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = sc.sc_kmeans(Y, n, R, w.k, restarts, iters, 4, None, lab, C)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(json.dumps({"workload": wl, "wide": wide, "pair": pair, "restarts": restarts, "max_iter": iters, "seconds": dt,
                      "inertia": res[0], "iters": res[1], "best": res[2]}), flush=True)
    out[(wide, pair)] = (lab.cpu().numpy(), C, res)
a = out[("1", "1")]
for key, b in out.items():
    print(key, "identical:", bool(np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]) and a[2] == b[2]))
