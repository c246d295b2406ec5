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
# 2-D decomposition: column groups x row blocks
# ---------------------------------------------------------------------------
#
# The columns of the signal block are independent filters (Y[:, q] = F^p R[:, q], PAPER.md
# Eq.(10) l.321 applies the same filter to every signal), so they shard across ranks with no
# exchange at all; only a row split needs the halo of T_j every step.  On graphs whose
# edges are spread at random (SBM) a row block's halo is nearly every other row, so the
# per-step halo traffic of a pure row partition grows with the number of ranks while its
# compute shrinks; splitting the columns first keeps each rank's gathered rows >= 128 bytes
# (the kernel is bound by gathered lines) and divides the halo traffic by the
# number of column groups.  Ranks [c * n_row, (c + 1) * n_row) form column group c; inside it
# they row-partition the graph exactly as above.

def grid_shape(world: int, R: int, min_cols: int = 32, col_groups: int | None = None):
    """(n_col_groups, n_row_blocks) for `world` ranks and R columns: the most column groups
    that divide world and R (in 4-column vectors) with >= min_cols columns each, unless
    col_groups is given."""
    if col_groups is not None:
        if world % col_groups or R % col_groups or (R // col_groups) % 4:
            raise ValueError(f"{col_groups} column groups do not divide world={world} and R={R} into 4-column sets")
        return col_groups, world // col_groups
    best = 1
    for c in range(1, world + 1):
        if world % c == 0 and R % c == 0 and (R // c) % 4 == 0 and R // c >= min_cols:
            best = c
    return best, world // best


def grid_coords(rank: int, world: int, n_col_groups: int):
    """(column group, row rank inside the group, global ranks of the group)."""
    n_row = world // n_col_groups
    c = rank // n_row
    return c, rank % n_row, list(range(c * n_row, (c + 1) * n_row))


def column_range(R: int, n_col_groups: int, c: int):
    """Columns [c0, c1) of column group c."""
    w = R // n_col_groups
    return c * w, (c + 1) * w


def make_row_groups(world: int, n_col_groups: int):
    """One process group per column group (collective: every rank calls it with the same
    arguments); returns the list indexed by column group (None for world 1)."""
    import torch.distributed as dist
    if world == 1:
        return [None]
    n_row = world // n_col_groups
    return [dist.new_group(list(range(c * n_row, (c + 1) * n_row))) for c in range(n_col_groups)]


def _cluster_partition(sc, parts, plans, comms, filt, k, R, order, jackson, n_probe, seed, restarts, max_iter,
                       normalize):
    """The accelerated spectral clustering (§4.1 steps 1-6) on a row partition, one
    library call per step: lambda_N (sc_dist_lambda_max), lambda~_k (sc_dist_estimate_lambda_k),
    the coefficients, the seeded signals of the ranks' rows (the same block as sc_cluster:
    stream 0, rows r0..r1 of the global block, permuted to local order), the filter (the
    caller's partitioned filter), the optional row normalisation, k-means over the ranks
    (sc_dist_kmeans, points in rank-major local order).  Random draws as sc_cluster.
    Returns (labels per rank in local order, info dict)."""
    import torch
    row0 = [p.r0 for p in parts]
    lmax = sc.sc_dist_lambda_max(plans, 60, 0.01, seed ^ 0x1A2B3C4D, row0)
    lam_k, count_k = sc.sc_dist_estimate_lambda_k(plans, k, lmax, order, True, n_probe, seed ^ 0x5E5E5E5E, row0,
                                                  40, 1e-4)
    d = sc.sc_cheby_coeffs(lam_k, lmax, order, jackson)
    Xs, Ys = [], []
    for p in parts:
        xb = torch.empty((p.n_local, R), dtype=torch.float32, device="cuda")
        sc.sc_random_signals_f32(p.n_local, R, p.r0, seed, 0, 0.0, xb)
        Xs.append(xb[torch.as_tensor(p.perm, device="cuda")].contiguous())
        Ys.append(torch.empty_like(Xs[-1]))
    filt(d, order, lmax, Xs, Ys)
    if normalize:
        for y in Ys:
            sc.sc_normalize_rows_f32(y, y.shape[0], R)
    labels = [torch.empty(p.n_local, dtype=torch.int32, device="cuda") for p in parts]
    inertia, iters, best = sc.sc_dist_kmeans(comms, Ys, R, k, restarts, max_iter, seed, None, labels)
    return labels, dict(lambda_max=lmax, lambda_k=lam_k, count_k=count_k, inertia=inertia, kmeans_iters=iters,
                        best_restart=best)


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
            dist.broadcast_object_list(uid, group=group, group_src=0)
        self.comm = _lib.sc_comm_init(uid[0], part.world, part.rank)
        self.plan = _lib.sc_dist_create(graph_handle, self.comm, part.n_interior, part.send_idx,
                                        np.asarray(part.send_counts, dtype=np.int64),
                                        np.asarray(part.recv_counts, dtype=np.int64))
        self.r0 = int(part.r0)   # counter offset of the rank's rows (start vector, probes)
        self.part = part

    def filter(self, d, order: int, lambda_max: float, X, Y):
        self._lib.sc_dist_filter_f32(self.plan, d, order, lambda_max, X.shape[1], X, Y)

    # PAPER.md §4.1 steps 1-2 on the partition (sc_dist_lambda_max / sc_dist_estimate_lambda_k):
    # halo exchange before every SpMV, inner products all-reduced; collective over the ranks
    def lambda_max(self, iters=60, margin=0.01, seed=0) -> float:
        return self._lib.sc_dist_lambda_max(self.plan, iters, margin, seed, [self.r0])

    def estimate_lambda_k(self, k, lambda_max, order, jackson=True, n_probe=32, seed=0, max_iter=40, rtol=1e-4):
        return self._lib.sc_dist_estimate_lambda_k(self.plan, k, lambda_max, order, jackson, n_probe, seed,
                                                   [self.r0], max_iter, rtol)

    def cluster(self, k, R, order, jackson=True, n_probe=32, seed=0, restarts=10, max_iter=100, normalize=False,
                filt=None):
        """PAPER.md §4.1 steps 1-6 for this rank (collective over the ranks; configs[4]'s
        "full pipeline including k-means"): see _cluster_partition.  filt: the rank's
        partitioned filter (default: this NCCL schedule)."""
        part = self.part

        def own_filter(d, order_, lmax, Xs, Ys):
            (filt or self.filter)(d, order_, lmax, Xs[0], Ys[0])
        return _cluster_partition(self._lib, [part], [self.plan], [self.comm], own_filter, k, R, order, jackson,
                                  n_probe, seed, restarts, max_iter, normalize)

    def close(self):
        if getattr(self, "plan", None):
            self._lib.sc_dist_free(self.plan)
            self.plan = None
        if getattr(self, "comm", None):
            self._lib.sc_comm_free(self.comm)
            self.comm = None


# ---------------------------------------------------------------------------
# fused peer-to-peer exchange (sc_p2p_*): descriptors and drivers
# ---------------------------------------------------------------------------

def p2p_descriptors(part: LocalPart, recv_counts_all):
    """Where each of this rank's rows goes in the peers' halos, CSR by local row.

    recv_counts_all[q][r] = rows rank q receives from rank r.  Rank q's halo is grouped by
    owner in ascending rank order and, inside an owner's block, in ascending global id --
    the order of the owner's send list to q -- so row send_idx[q][j] lands at q's halo slot
    sum(recv_counts_all[q][:rank]) + j.  Returns (sd_ptr, sd_row, sd_peer, sd_slot)."""
    r, nl = part.rank, part.n_local
    rows, peers, slots = [], [], []
    so = 0
    for q in range(part.world):
        cnt = int(part.send_counts[q])
        if q == r or cnt == 0:
            so += cnt
            continue
        base = int(sum(recv_counts_all[q][:r]))
        rows.append(np.asarray(part.send_idx[so:so + cnt], dtype=np.int64))
        peers.append(np.full(cnt, q, dtype=np.int32))
        slots.append(base + np.arange(cnt, dtype=np.int64))
        so += cnt
    if rows:
        row = np.concatenate(rows)
        peer = np.concatenate(peers)
        slot = np.concatenate(slots)
        o = np.argsort(row, kind="stable")
        row, peer, slot = row[o], peer[o], slot[o]
    else:
        row = np.zeros(0, np.int64)
        peer = np.zeros(0, np.int32)
        slot = np.zeros(0, np.int64)
    ptr = np.zeros(nl + 1, dtype=np.int64)
    np.cumsum(np.bincount(row, minlength=nl), out=ptr[1:])
    return ptr, row, peer, slot


class P2PFilter:
    """One rank of the fused-exchange filter (one process per GPU): descriptors from the
    all-gathered receive counts, CUDA IPC handles of every rank's T buffers exchanged with
    torch.distributed, then sc_p2p_filter_f32 per call."""

    def __init__(self, part: LocalPart, graph_handle, n_global: int, max_R: int, group=None):
        import torch.distributed as dist
        from . import _lib as sc
        self.part, self.sc = part, sc
        w = part.world
        rc_all, nl_all, hs = [list(part.recv_counts)], [int(part.n_local)], [None]
        if w > 1:
            rc_all, nl_all, hs = [None] * w, [None] * w, [None] * w
            dist.all_gather_object(rc_all, list(part.recv_counts), group=group)
            dist.all_gather_object(nl_all, int(part.n_local), group=group)
        sd = p2p_descriptors(part, rc_all)
        self.handle = sc.sc_p2p_create(graph_handle, w, part.rank, n_global, *sd, nl_all, max_R)
        if w > 1:
            dist.all_gather_object(hs, sc.sc_p2p_export(self.handle), group=group)
            for q in range(w):
                if q != part.rank:
                    sc.sc_p2p_import(self.handle, q, hs[q])
            dist.barrier(group=group)

    def filter(self, d, order, lambda_max, X, Y, stream=None):
        self.sc.sc_p2p_filter_f32(self.handle, d, order, lambda_max, X.shape[1], X, Y, stream)

    def close(self):
        if self.handle:
            self.sc.sc_p2p_free(self.handle)
            self.handle = None


class P2PGroup:
    """All ranks of a row partition in one process on one GPU (single-GPU emulation of the
    fused exchange, tests): sc_p2p_filter_group_f32 runs the same kernels in dependency
    order on one stream."""

    def __init__(self, row_ptr, col_idx, values, n: int, world: int, max_R: int):
        from . import _lib as sc
        from . import Graph
        self.sc = sc
        parts = [local_part(row_ptr, col_idx, values, n, r, world) for r in range(world)]
        halos = [p.halo_gid for p in parts]
        self.parts = [send_lists_from_halos(p, halos) for p in parts]
        rc_all = [p.recv_counts for p in self.parts]
        nl_all = [p.n_local for p in self.parts]
        self.graphs = [Graph(p.n_local, p.row_ptr, p.col_idx, p.values, n_cols=p.n_local + p.n_halo)
                       for p in self.parts]
        self.handles = [sc.sc_p2p_create(self.graphs[r].handle, world, r, n, *p2p_descriptors(self.parts[r], rc_all),
                                         nl_all, max_R) for r in range(world)]
        for a in range(world):
            for b in range(world):
                if a != b:
                    sc.sc_p2p_link_local(self.handles[a], self.handles[b])
        # the same partition as sc_dist plans on local (emulation) communicators: the lambda
        # estimates and the distributed k-means of the pipeline
        self.comms = [sc.sc_comm_local(world, r) for r in range(world)]
        self.plans = [sc.sc_dist_create(self.graphs[r].handle, self.comms[r], p.n_interior, p.send_idx,
                                        np.asarray(p.send_counts, dtype=np.int64),
                                        np.asarray(p.recv_counts, dtype=np.int64))
                      for r, p in enumerate(self.parts)]
        self.world = world

    def filter(self, d, order, lambda_max, Xs, Ys, stream=None):
        self.sc.sc_p2p_filter_group_f32(self.handles, d, order, lambda_max, Xs[0].shape[1], Xs, Ys, stream)

    def cluster(self, k, R, order, jackson=True, n_probe=32, seed=0, restarts=10, max_iter=100, normalize=False):
        """PAPER.md §4.1 steps 1-6 on the partition (every rank held here): see _cluster_partition."""
        return _cluster_partition(self.sc, self.parts, self.plans, self.comms, self.filter, k, R, order, jackson,
                                  n_probe, seed, restarts, max_iter, normalize)

    def close(self):
        for h in self.handles:
            self.sc.sc_p2p_free(h)
        self.handles = []
        for pl in getattr(self, "plans", []):
            self.sc.sc_dist_free(pl)
        self.plans = []
        for c in getattr(self, "comms", []):
            self.sc.sc_comm_free(c)
        self.comms = []
        for g in self.graphs:
            g.close()
