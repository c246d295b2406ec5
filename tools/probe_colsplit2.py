"""Column-split emulation (DESIGN.md §0(f) item 1), GPU box: one launch over a random
graph (N = 10^6, 20 nnz/row, uniform columns) vs two launches over its two column halves
(10 nnz/row each, 64 MB gathered table each), the first writing a partial block that the
second reads back in place of T_{s-1}."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1509_08863_b200 as sc

N, DEG, R = 1_000_000, 20, 32
rng = np.random.default_rng(7)
def load(lo, hi, deg):
    col = np.sort(rng.integers(lo, hi, size=(N, deg), dtype=np.int32), axis=1).reshape(-1)
    rp = np.arange(0, N * deg + 1, deg, dtype=np.int64)
    return sc.sc_graph_load(N, N, N * deg, rp, col, None)
full = load(0, N, DEG)
h0 = load(0, N // 2, DEG // 2)
h1 = load(N // 2, N, DEG // 2)
T0, T1, T2, P = (torch.randn(N, R, device="cuda") for _ in range(4))
def st(h, tprev, tnext):
    sc.sc_cheb_step_f32(h, 0, N, R, tprev, R, T1, R, tnext, R, None, R, 0.1, -2.0, -1.0 if tprev is not None else 0.0,
                        0, 0, 0, 0)
def timeit(fn, reps=50):
    for _ in range(5): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return round(e0.elapsed_time(e1) * 1000 / reps, 1)
out = {"one_launch_us": timeit(lambda: st(full, T0, T2)),
       "half_A_us": timeit(lambda: st(h0, None, P)),
       "half_B_us": timeit(lambda: st(h1, P, T2))}
out["split_pair_us"] = timeit(lambda: (st(h0, None, P), st(h1, P, T2)))
print(json.dumps(out))
