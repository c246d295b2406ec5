"""Per-call wall times of repeated C-ABI calls (GPU box): looks for sporadic host-side stalls."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gc
import torch
if os.environ.get("NO_GC"):
    gc.disable()
import paper_1509_08863_b200 as sc
from scinputs import configs

wl = sys.argv[1] if len(sys.argv) > 1 else "c3_sbm1m"
w = configs.WORKLOADS[wl]
g = configs.build_graph(wl, cache=True)
G = sc.Graph.from_csr(g)
n, R = g.n, w.R
lmax = 2.0 * G.info()[3]
Y = torch.empty((n, R), dtype=torch.float32, device="cuda")
lab = torch.empty(n, dtype=torch.int32, device="cuda")
out = {"filter": [], "kmeans": [], "lambda_k": []}
for it in range(int(sys.argv[2]) if len(sys.argv) > 2 else 6):
    for name, fn in (("filter", lambda: sc.sc_filter_lowpass_f32(G.handle, 0.005 * lmax, lmax, w.order, w.jackson, R, 3, None, Y)),
                     ("lambda_k", lambda: sc.sc_estimate_lambda_k(G.handle, w.k, lmax, w.order, True, 32, 2, 40, 1e-4)),
                     ("kmeans", lambda: sc.sc_kmeans(Y, n, R, w.k, 1, 20, 4, None, lab))):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        c0 = time.process_time()
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        out[name].append((round(time.perf_counter() - t0, 4), round(e0.elapsed_time(e1) / 1e3, 4),
                          round(time.process_time() - c0, 4)))
print(json.dumps(out))
