"""Row-partitioned multi-GPU Chebyshev filter (one process per GPU).

BASELINE.json north_star: "the graph is row-partitioned.  Each recurrence step
exchanges the needed rows of T_j over NVLink with NCCL ... as a halo-only
exchange, overlapped with the interior SpMM."

Each rank owns a contiguous block of rows [r0, r1) of W.  Its local CSR is
renumbered so that columns [0, n_local) are its own rows and columns
[n_local, n_local + n_halo) are the remote rows it reads (the halo), in
ascending global id.  Local rows are permuted so that *interior* rows (no halo
neighbour) come first: per step the halo of T_s is exchanged with
``all_to_all_single`` on the process group while the step kernel runs over the
interior rows; the boundary rows run after the exchange lands.

The arithmetic of every step runs in ``sc_cheb_step_f32`` (CUDA) on GPU ranks.
Host logic here (partitioning, halo lists, exchange, step schedule) is
backend-agnostic: with the ``gloo`` backend and a CPU step function it is
tested on CPU (tests/test_dist_cpu.py).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


# ---------------------------------------------------------------------------
# partitioning and halo lists
# ---------------------------------------------------------------------------

def partition_rows(n: int, world: int):
    """Contiguous, balanced row blocks: list of (r0, r1) per rank."""
    base, extra = divmod(n, world)
    out, r = [], 0
    for q in range(world):
        m = base + (1 if q < extra else 0)
        out.append((r, r + m))
        r += m
    return out


@dataclass
class LocalPart:
    rank: int
    world: int
    r0: int
    r1: int
    n_local: int
    n_halo: int
    row_ptr: np.ndarray        # int64 [n_local+1], rows in local (interior-first) order
    col_idx: np.ndarray        # int32, renumbered columns
    values: np.ndarray | None
    perm: np.ndarray           # local position -> original local row (r - r0)
    n_interior: int
    halo_gid: np.ndarray       # global ids of halo rows (ascending)
    recv_counts: list          # rows received from each peer (halo is grouped by owner, ascending)
    send_idx: np.ndarray       # local positions (permuted order) to send, grouped by peer
    send_counts: list


def local_part(row_ptr, col_idx, values, n: int, rank: int, world: int) -> LocalPart:
    """Build rank's renumbered local CSR and its halo receive list from the global CSR.
    (Send lists need the peers' halos: see ``exchange_send_lists``.)"""
    parts = partition_rows(n, world)
    r0, r1 = parts[rank]
    nl = r1 - r0
    rp = np.asarray(row_ptr[r0:r1 + 1], dtype=np.int64) - int(row_ptr[r0])
    cols = np.asarray(col_idx[row_ptr[r0]:row_ptr[r1]], dtype=np.int64)
    vals = None if values is None else np.asarray(values[row_ptr[r0]:row_ptr[r1]], dtype=np.float32)
    remote = (cols < r0) | (cols >= r1)
    halo_gid = np.unique(cols[remote])
    # interior rows: no remote neighbour
    rows_of = np.repeat(np.arange(nl), np.diff(rp))
    has_remote = np.zeros(nl, dtype=bool)
    has_remote[rows_of[remote]] = True
    perm = np.concatenate([np.nonzero(~has_remote)[0], np.nonzero(has_remote)[0]]).astype(np.int64)
    inv = np.empty(nl, dtype=np.int64)
    inv[perm] = np.arange(nl)
    # renumber columns: own rows -> permuted local position, remote -> nl + halo position
    newc = np.empty_like(cols)
    newc[~remote] = inv[cols[~remote] - r0]
    newc[remote] = nl + np.searchsorted(halo_gid, cols[remote])
    # permute rows
    deg = np.diff(rp)[perm]
    prp = np.zeros(nl + 1, dtype=np.int64)
    np.cumsum(deg, out=prp[1:])
    order = np.concatenate([np.arange(rp[p], rp[p + 1]) for p in perm]) if nl else np.zeros(0, np.int64)
    pc = newc[order].astype(np.int32)
    pv = None if vals is None else vals[order]
    owner = np.searchsorted([p[1] for p in parts], halo_gid, side="right")
    recv_counts = [int(np.sum(owner == q)) for q in range(world)]
    return LocalPart(rank, world, r0, r1, nl, int(halo_gid.size), prp, pc, pv, perm,
                     int(np.sum(~has_remote)), halo_gid, recv_counts, np.zeros(0, np.int64), [0] * world)


def exchange_send_lists(part: LocalPart, group=None) -> LocalPart:
    """Every rank learns which of its rows each peer needs (all_gather of halo lists)."""
    import torch.distributed as dist
    halos = [None] * part.world
    dist.all_gather_object(halos, part.halo_gid, group=group)
    return send_lists_from_halos(part, halos)


def send_lists_from_halos(part: LocalPart, halos) -> LocalPart:
    """Fill part.send_idx / send_counts from every rank's halo list (halos[q] = global ids
    rank q reads).  Rows for peer q are sent in ascending global id, which is the order
    of q's halo block for this owner."""
    inv = np.empty(part.n_local, dtype=np.int64)
    inv[part.perm] = np.arange(part.n_local)
    send, counts = [], []
    for q in range(part.world):
        if q == part.rank:
            counts.append(0)
            continue
        h = np.asarray(halos[q])
        mine = h[(h >= part.r0) & (h < part.r1)]
        send.append(inv[mine - part.r0])
        counts.append(int(mine.size))
    part.send_idx = np.concatenate(send) if send else np.zeros(0, np.int64)
    part.send_counts = counts
    return part


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
    from . import _lib

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


class NcclFilter:
    """The whole row-partitioned filter inside the library (``sc_dist_filter_f32``): per
    step the halo of T_s is exchanged with NCCL send/recv on the communicator's stream
    while the interior rows' fused step runs; the boundary rows follow.  Same schedule as
    ``run_filter`` without any per-step Python.  X and Y are in the plan's local
    (interior-first) row order: ``X_local[torch.as_tensor(part.perm)]``."""

    def __init__(self, part: LocalPart, graph_handle, group=None):
        from . import _lib
        self._lib = _lib
        uid = [_lib.sc_nccl_unique_id() if part.rank == 0 else None]
        if part.world > 1:
            import torch.distributed as dist
            dist.broadcast_object_list(uid, src=0, group=group)
        self.comm = _lib.sc_comm_init(uid[0], part.world, part.rank)
        self.plan = _lib.sc_dist_create(graph_handle, self.comm, part.n_interior, part.send_idx,
                                        np.asarray(part.send_counts, dtype=np.int64),
                                        np.asarray(part.recv_counts, dtype=np.int64))

    def filter(self, d, order: int, lambda_max: float, X, Y):
        self._lib.sc_dist_filter_f32(self.plan, d, order, lambda_max, X.shape[1], X, Y)

    def close(self):
        if getattr(self, "plan", None):
            self._lib.sc_dist_free(self.plan)
            self.plan = None
        if getattr(self, "comm", None):
            self._lib.sc_comm_free(self.comm)
            self.comm = None
