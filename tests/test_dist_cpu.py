"""Row-partitioned multi-process filter on CPU (gloo, world_size 2 and 3).

Exercises the host logic of paper_1509_08863_b200.dist -- partitioning, column
renumbering, interior-first row permutation, halo send/recv lists, the
all_to_all halo exchange and the fused-step schedule -- with a CPU step
function, and compares the gathered result with the oracle on the whole graph.
"""

import os
import socket

import numpy as np
import pytest
import scipy.sparse as sp
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import scinputs
from oracle import chebyshev, laplacian

import dist_reference as dref


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _cpu_step_fn(part):
    W = sp.csr_matrix((np.ones(part.col_idx.size) if part.values is None else part.values.astype(np.float64),
                       part.col_idx, part.row_ptr), shape=(part.n_local, part.n_local + part.n_halo))
    s = np.asarray(W.sum(axis=1)).ravel()

    def fn(rb, re, T_prev, T_cur, T_next, Y, st):
        if re <= rb:
            return
        Tc = T_cur.numpy().astype(np.float64)
        acc = W[rb:re] @ Tc
        own = Tc[rb:re]
        prv = T_prev.numpy()[rb:re].astype(np.float64) if T_prev is not None else 0.0
        tn = st["a"] * (s[rb:re, None] * own - acc) + st["b_cur"] * own + st["b_prev"] * prv
        if T_next is not None:
            T_next[rb:re] = torch.from_numpy(tn)
        if st["y_mode"]:
            upd = st["cy_prev"] * prv + st["cy_cur"] * own + st["cy_next"] * tn
            if st["y_mode"] == 1:
                Y[rb:re] = torch.from_numpy(np.asarray(upd + 0.0 * own))
            else:
                Y[rb:re] += torch.from_numpy(np.asarray(upd + 0.0 * own))
    return fn


def _worker(rank, world, port, gspec, R, order, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1509_08863_b200 import dist as pdist
        g = scinputs.sbm(**gspec)
        part = pdist.local_part(g.row_ptr, g.col_idx, g.values, g.n, rank, world)
        part = pdist.exchange_send_lists(part)
        lmax = 2.0 * float(g.degrees().max())
        d = chebyshev.filter_coeffs(0.15 * lmax, lmax, order, True)
        X = torch.from_numpy(scinputs.gaussian_block(5, g.n, R).astype(np.float64))
        Xl = X[part.r0:part.r1].contiguous()
        Y = dref.run_filter(part, _cpu_step_fn(part), d, order, lmax, Xl)
        parts = [None] * world
        dist.all_gather_object(parts, (part.r0, part.r1, Y.numpy(), part.n_interior, part.n_halo))
        if rank == 0:
            Yfull = np.zeros((g.n, R))
            for r0, r1, y, _, _ in parts:
                Yfull[r0:r1] = y
            Yo = chebyshev.cheb_filter(laplacian.laplacian(g), X.numpy(), d, lmax)
            err = np.linalg.norm(Yfull - Yo) / np.linalg.norm(Yo)
            q.put((err, [(p[3], p[4]) for p in parts]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,eps", [(2, 0.05), (3, 0.0)])
def test_distributed_filter_gloo(world, eps):
    gspec = dict(n=1200, k=4, avg_degree=8, eps=eps, seed=3)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, gspec, 8, 20, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(180)
        assert p.exitcode == 0
    err, info = q.get(timeout=10)
    assert err < 1e-12
    if eps == 0.0:
        # disconnected communities aligned with the partition -> no halo for SBM blocks
        # fully owned by one rank; interior rows exist on every rank
        assert all(ni > 0 for ni, _ in info)


def test_partition_and_schedule_pure():
    from paper_1509_08863_b200 import dist as pdist
    assert pdist.partition_rows(10, 3) == [(0, 4), (4, 7), (7, 10)]
    # schedule adds every T_j to Y exactly once with its coefficient
    for order in [1, 2, 3, 4, 5, 9, 10]:
        d = np.arange(1, order + 2, dtype=float)
        seen = np.zeros(order + 1)
        for st in dref.step_schedule(order, d, 2.0):
            s = st["s"]
            if st["y_mode"]:
                if s >= 1:
                    seen[s - 1] += st["cy_prev"]
                seen[s] += st["cy_cur"]
                seen[s + 1] += st["cy_next"]
        assert np.array_equal(seen, d)


# ---------------------------------------------------------------------------
# fused peer-to-peer exchange: the descriptors a rank's step kernel uses to store its
# boundary rows straight into the peers' halos (sc_p2p_*)
# ---------------------------------------------------------------------------

def _p2p_worker(rank, world, port, gspec, R, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1509_08863_b200 import dist as pdist
        g = scinputs.sbm(**gspec)
        part = pdist.exchange_send_lists(pdist.local_part(g.row_ptr, g.col_idx, g.values, g.n, rank, world))
        rc_all = [None] * world
        dist.all_gather_object(rc_all, list(part.recv_counts))
        ptr, row, peer, slot = pdist.p2p_descriptors(part, rc_all)
        X = scinputs.gaussian_block(9, g.n, R)
        T_local = X[part.r0:part.r1][part.perm]            # this rank's rows, local (permuted) order
        out = [(int(peer[e]), int(slot[e]), T_local[int(row[e])]) for e in range(row.size)]
        sent = [None] * world
        dist.all_gather_object(sent, out)
        halo = np.full((part.n_halo, R), np.nan, dtype=X.dtype)
        writes = np.zeros(part.n_halo, dtype=int)
        for lst in sent:
            for pq, sl, v in lst:
                if pq == rank:
                    halo[sl] = v
                    writes[sl] += 1
        ok = (np.all(writes == 1) and np.array_equal(halo, X[part.halo_gid])
              and np.all(np.diff(ptr) >= 0) and ptr[-1] == row.size and np.all(np.diff(row) >= 0)
              and np.all(peer != rank))
        q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_p2p_descriptors_fill_every_halo_exactly_once_gloo(world):
    gspec = dict(n=900, k=3, avg_degree=8, eps=0.1, seed=4)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_p2p_worker, args=(r, world, port, gspec, 4, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(180)
        assert p.exitcode == 0
    res = dict(q.get(timeout=10) for _ in range(world))
    assert all(res[r] for r in range(world))


@pytest.mark.parametrize("world", [1, 2, 4, 5])
def test_p2p_scatter_reference_reproduces_halos(world):
    from paper_1509_08863_b200 import dist as pdist
    g = scinputs.sbm(700, 5, 6, 0.2, seed=6)
    parts = [pdist.local_part(g.row_ptr, g.col_idx, g.values, g.n, r, world) for r in range(world)]
    halos = [p.halo_gid for p in parts]
    parts = [pdist.send_lists_from_halos(p, halos) for p in parts]
    X = scinputs.gaussian_block(2, g.n, 3)
    T_locals = [X[p.r0:p.r1][p.perm] for p in parts]
    got = dref.p2p_scatter_reference(parts, T_locals)
    for p, h in zip(parts, got):
        assert np.array_equal(h, X[p.halo_gid])


# ---------------------------------------------------------------------------
# 2-D decomposition: column groups (no exchange) x row blocks (halo exchange inside the
# group's own process group)
# ---------------------------------------------------------------------------

def _grid_worker(rank, world, port, gspec, R, order, n_cg, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1509_08863_b200 import dist as pdist
        g = scinputs.sbm(**gspec)
        n_cg2, n_row = pdist.grid_shape(world, R, min_cols=4, col_groups=n_cg)
        cgrp, rrank, members = pdist.grid_coords(rank, world, n_cg2)
        c0, c1 = pdist.column_range(R, n_cg2, cgrp)
        groups = pdist.make_row_groups(world, n_cg2)
        part = pdist.local_part(g.row_ptr, g.col_idx, g.values, g.n, rrank, n_row)
        part = (pdist.exchange_send_lists(part, group=groups[cgrp]) if n_row > 1
                else pdist.send_lists_from_halos(part, [part.halo_gid]))
        lmax = 2.0 * float(g.degrees().max())
        d = chebyshev.filter_coeffs(0.15 * lmax, lmax, order, True)
        X = torch.from_numpy(scinputs.gaussian_block(5, g.n, R).astype(np.float64))
        Xl = X[part.r0:part.r1, c0:c1].contiguous()
        Y = dref.run_filter(part, _cpu_step_fn(part), d, order, lmax, Xl, group=groups[cgrp])
        outs = [None] * world
        dist.all_gather_object(outs, (part.r0, part.r1, c0, c1, Y.numpy(), rank in members))
        if rank == 0:
            Yfull = np.full((g.n, R), np.nan)
            for r0, r1, a, b, y, _ in outs:
                assert np.all(np.isnan(Yfull[r0:r1, a:b]))   # every block written exactly once
                Yfull[r0:r1, a:b] = y
            Yo = chebyshev.cheb_filter(laplacian.laplacian(g), X.numpy(), d, lmax)
            err = np.linalg.norm(Yfull - Yo) / np.linalg.norm(Yo)
            q.put((err, (n_cg2, n_row), all(o[5] for o in outs)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n_cg", [(4, 2), (2, 2)])
def test_column_x_row_grid_filter_gloo(world, n_cg):
    gspec = dict(n=1000, k=4, avg_degree=8, eps=0.1, seed=7)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_grid_worker, args=(r, world, port, gspec, 8, 15, n_cg, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(180)
        assert p.exitcode == 0
    err, shape, member_ok = q.get(timeout=10)
    assert shape == (n_cg, world // n_cg) and member_ok
    assert err < 1e-12


def test_grid_shape_rule():
    from paper_1509_08863_b200 import dist as pdist
    # configs[3] (R = 64): 2 column groups of 32 once there are >= 2 ranks
    assert [pdist.grid_shape(w, 64) for w in (1, 2, 4, 8)] == [(1, 1), (2, 1), (2, 2), (2, 4)]
    # configs[4] (R = 96): 2 groups of 48 (3 does not divide 2, 4 or 8; 4 groups would be 24 wide)
    assert [pdist.grid_shape(w, 96) for w in (1, 2, 4, 8)] == [(1, 1), (2, 1), (2, 2), (2, 4)]
    # R too narrow for two >= 32-column groups: pure row partition
    assert pdist.grid_shape(8, 48) == (1, 8)
    assert pdist.grid_shape(8, 64, col_groups=1) == (1, 8)
    assert pdist.grid_shape(8, 64, col_groups=4) == (4, 2)
    with pytest.raises(ValueError):
        pdist.grid_shape(8, 64, col_groups=3)
    assert pdist.grid_coords(5, 8, 2) == (1, 1, [4, 5, 6, 7])
    assert pdist.column_range(64, 2, 1) == (32, 64)
