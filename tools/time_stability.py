"""Stability scan gamma(k) on a workload (GPU box): sc_stability over [k_min, k_max] with
J redraws (configs[2]: k in [10, 30], J = 10, R = 48, p = 150)."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1509_08863_b200 as sc
from scinputs import configs

wl = sys.argv[1] if len(sys.argv) > 1 else "c2_sbm100k"
kmin, kmax, J = (int(x) for x in (sys.argv[2:5] if len(sys.argv) > 4 else (10, 30, 10)))
restarts = int(sys.argv[5]) if len(sys.argv) > 5 else 5
w = configs.WORKLOADS[wl]
g = configs.build_graph(wl, cache=True)
G = sc.Graph.from_csr(g)
reps = int(os.environ.get("REPS", "1"))
for rep in range(reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    gam, lk = sc.sc_stability(G.handle, kmin, kmax, J, w.R, w.order, True, 32, 11, restarts, 100)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    if rep < reps - 1:
        print(json.dumps({"rep": rep, "seconds": dt}), flush=True)
ks = list(range(kmin, kmax + 1))
print(json.dumps({"workload": wl, "k_range": [kmin, kmax], "J": J, "R": w.R, "order": w.order, "restarts": restarts,
                  "seconds": dt, "k_star": ks[int(np.argmax(gam))], "gamma": [round(float(x), 4) for x in gam],
                  "lambda_k": [float(x) for x in lk]}))
