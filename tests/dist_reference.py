"""Reference schedules of the row-partitioned filter, in Python (TEST SCAFFOLDING).

Moved out of the product package (VERDICT r01 "test scaffolding lives in the product"): a
per-step Python driver of the partitioned filter with a torch.distributed halo exchange
(run_filter, HaloExchange; exercised with gloo on CPU), the per-step schedule, the C-ABI step
function, and the host model of the fused peer-store exchange (p2p_scatter_reference).
"""

from __future__ import annotations

import numpy as np

from paper_1509_08863_b200.dist import LocalPart, p2p_descriptors  # noqa: F401


# ---------------------------------------------------------------------------
# step schedule (coefficients per launch)
# ---------------------------------------------------------------------------

def step_schedule(order: int, d, lambda_max: float):
    """Per-step arguments of the fused recurrence: T_{s+1} = a L T_s + b_cur T_s +
    b_prev T_{s-1}; Y is updated when three terms are pending or at the last step."""
    added = -1
    for s in range(order):
        last = s == order - 1
        st = dict(s=s, a=(2.0 if s == 0 else 4.0) / lambda_max, b_cur=-1.0 if s == 0 else -2.0,
                  b_prev=0.0 if s == 0 else -1.0, cy_prev=0.0, cy_cur=0.0, cy_next=0.0, y_mode=0,
                  store_next=not last)
        if last or (s + 1) - added == 3:
            st["cy_prev"] = float(d[s - 1]) if (s >= 1 and added < s - 1) else 0.0
            st["cy_cur"] = float(d[s]) if added < s else 0.0
            st["cy_next"] = float(d[s + 1])
            st["y_mode"] = 1 if added == -1 else 2
            added = s + 1
        yield st


# ---------------------------------------------------------------------------
# driver
# ---------------------------------------------------------------------------

class HaloExchange:
    """all_to_all_single of the halo rows of a (n_local + n_halo) x R block."""

    def __init__(self, part: LocalPart, R: int, device, dtype, group=None):
        import torch
        self.part, self.group, self.R = part, group, R
        self.send_idx = torch.as_tensor(part.send_idx, dtype=torch.int64, device=device)
        self.send_buf = torch.empty((int(part.send_idx.size), R), dtype=dtype, device=device)
        self.recv_buf = torch.empty((part.n_halo, R), dtype=dtype, device=device)

    def start(self, T):
        import torch
        import torch.distributed as dist
        if self.part.world == 1:
            return None
        torch.index_select(T[: self.part.n_local], 0, self.send_idx, out=self.send_buf)
        return dist.all_to_all_single(self.recv_buf, self.send_buf, self.part.recv_counts, self.part.send_counts,
                                      group=self.group, async_op=True)

    def finish(self, work, T):
        if work is None:
            return
        work.wait()
        T[self.part.n_local:].copy_(self.recv_buf)


def run_filter(part: LocalPart, step_fn, d, order: int, lambda_max: float, X_local, group=None):
    """Y_local = sum_j d_j T_j X restricted to this rank's rows (original local order).

    step_fn(row_begin, row_end, T_prev, T_cur, T_next, Y, st) runs one fused step on
    local rows [row_begin, row_end) of the permuted order (GPU: sc_cheb_step_f32)."""
    import torch
    nl, nh = part.n_local, part.n_halo
    R = X_local.shape[1]
    dev, dt = X_local.device, X_local.dtype
    perm = torch.as_tensor(part.perm, dtype=torch.int64, device=dev)
    T0 = torch.zeros((nl + nh, R), dtype=dt, device=dev)
    T0[:nl] = X_local.index_select(0, perm)
    bufs = [torch.zeros((nl + nh, R), dtype=dt, device=dev) for _ in range(2)]   # T_j in bufs[j & 1]
    Y = torch.empty((nl, R), dtype=dt, device=dev)
    ex = HaloExchange(part, R, dev, dt, group)
    for st in step_schedule(order, d, lambda_max):
        s = st["s"]
        T_cur = T0 if s == 0 else bufs[s & 1]
        T_prev = None if s == 0 else (T0 if s == 1 else bufs[(s - 1) & 1])
        T_next = bufs[(s + 1) & 1] if st["store_next"] else None
        work = ex.start(T_cur)
        step_fn(0, part.n_interior, T_prev, T_cur, T_next, Y, st)
        ex.finish(work, T_cur)
        step_fn(part.n_interior, nl, T_prev, T_cur, T_next, Y, st)
    out = torch.empty_like(Y)
    out[perm] = Y
    return out


def cuda_step_fn(handle):
    """step_fn backed by the C ABI (fp32, device buffers)."""
    from paper_1509_08863_b200 import _lib

    def fn(rb, re, T_prev, T_cur, T_next, Y, st):
        if re <= rb:
            return
        R = T_cur.shape[1]
        _lib.sc_cheb_step_f32(handle, rb, re, R, T_prev, R, T_cur, R, T_next, R, Y, R, st["a"], st["b_cur"],
                              st["b_prev"], st["cy_prev"], st["cy_cur"], st["cy_next"], st["y_mode"])
    return fn


def filter_local_steps(handle, d, order, lambda_max, X, row_split=None):
    """Single-GPU use of the per-step entry point over several row ranges (tests)."""
    import torch
    n, R = X.shape
    split = list(row_split) if row_split else [0, n]
    fn = cuda_step_fn(handle)
    bufs = [torch.zeros_like(X) for _ in range(2)]
    Y = torch.empty_like(X)
    for st in step_schedule(order, d, lambda_max):
        s = st["s"]
        T_cur = X if s == 0 else bufs[s & 1]
        T_prev = None if s == 0 else (X if s == 1 else bufs[(s - 1) & 1])
        T_next = bufs[(s + 1) & 1] if st["store_next"] else None
        for a, b in zip(split[:-1], split[1:]):
            fn(a, b, T_prev, T_cur, T_next, Y, st)
    return Y




def p2p_scatter_reference(parts, T_locals):
    """Host model of the fused exchange (tests): every rank's descriptors applied to its
    local rows; returns each rank's halo block."""
    rc_all = [p.recv_counts for p in parts]
    halos = [np.zeros((p.n_halo,) + T_locals[p.rank].shape[1:], dtype=T_locals[p.rank].dtype) for p in parts]
    for p in parts:
        ptr, row, peer, slot = p2p_descriptors(p, rc_all)
        for e in range(row.size):
            halos[int(peer[e])][int(slot[e])] = T_locals[p.rank][int(row[e])]
    return halos


