"""ctypes binding of libsc_b200.so -- argument marshalling only.

Every function here has the name of the C entry point it calls
(include/sc_b200.h) and does nothing but convert Python arguments (torch
tensors, numpy arrays, scalars) into pointers and sizes, call the library and
turn a non-zero status into an exception.  All arithmetic of the method runs in
the library's CUDA kernels; there is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SC_B200_LIB", os.path.join(_HERE, "libsc_b200.so"))

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"libsc_b200.so not found at {LIB_PATH}: build it with `python native_build.py` "
        "(or __graft_entry__.build()). There is no CPU fallback.")

_lib = ctypes.CDLL(LIB_PATH)

c_i64 = ctypes.c_int64
c_i32 = ctypes.c_int
c_u64 = ctypes.c_uint64
c_dbl = ctypes.c_double
c_vp = ctypes.c_void_p
P = ctypes.POINTER


def _sig(name, *args):
    f = getattr(_lib, name)
    f.restype = ctypes.c_int
    f.argtypes = list(args)
    return f


_lib.sc_last_error.restype = ctypes.c_char_p
_lib.sc_version.restype = ctypes.c_int

_F = {
    "sc_graph_load": _sig("sc_graph_load", c_i64, c_i64, c_i64, c_vp, c_vp, c_vp, P(c_vp)),
    "sc_graph_free": _sig("sc_graph_free", c_vp),
    "sc_graph_info": _sig("sc_graph_info", c_vp, P(c_i64), P(c_i64), P(c_i64), P(c_dbl)),
    "sc_graph_strengths": _sig("sc_graph_strengths", c_vp, c_vp, c_vp),
    "sc_lambda_max": _sig("sc_lambda_max", c_vp, c_i32, c_dbl, c_u64, P(c_dbl), c_vp),
    "sc_cheby_coeffs": _sig("sc_cheby_coeffs", c_dbl, c_dbl, c_i32, c_i32, c_vp),
    "sc_filter_order": _sig("sc_filter_order", c_dbl, c_dbl, c_i32, c_dbl, c_i32, c_i32, P(c_i32), P(c_dbl), c_vp),
    "sc_random_signals_f32": _sig("sc_random_signals_f32", c_i64, c_i32, c_i64, c_u64, c_i32, c_dbl, c_vp, c_vp),
    "sc_random_signals_f64": _sig("sc_random_signals_f64", c_i64, c_i32, c_i64, c_u64, c_i32, c_dbl, c_vp, c_vp),
    "sc_filter_apply_f32": _sig("sc_filter_apply_f32", c_vp, c_vp, c_i32, c_dbl, c_i32, c_vp, c_vp, c_vp),
    "sc_filter_apply_f64": _sig("sc_filter_apply_f64", c_vp, c_vp, c_i32, c_dbl, c_i32, c_vp, c_vp, c_vp),
    "sc_filter_lowpass_f32": _sig("sc_filter_lowpass_f32", c_vp, c_dbl, c_dbl, c_i32, c_i32, c_i32, c_u64, c_vp,
                                  c_vp, c_vp),
    "sc_filter_lowpass_f64": _sig("sc_filter_lowpass_f64", c_vp, c_dbl, c_dbl, c_i32, c_i32, c_i32, c_u64, c_vp,
                                  c_vp, c_vp),
    "sc_cheb_step_f32": _sig("sc_cheb_step_f32", c_vp, c_i64, c_i64, c_i32, c_vp, c_i64, c_vp, c_i64, c_vp, c_i64,
                             c_vp, c_i64, c_dbl, c_dbl, c_dbl, c_dbl, c_dbl, c_dbl, c_i32, c_vp),
    "sc_cheb_moments": _sig("sc_cheb_moments", c_vp, c_dbl, c_i32, c_i32, c_u64, c_vp, c_vp, c_vp),
    "sc_eigencount_from_moments": _sig("sc_eigencount_from_moments", c_vp, c_i32, c_dbl, c_dbl, c_i32, P(c_dbl)),
    "sc_estimate_lambda_k": _sig("sc_estimate_lambda_k", c_vp, c_i32, c_dbl, c_i32, c_i32, c_i32, c_u64, c_i32, c_dbl,
                                 P(c_dbl), P(c_dbl), c_vp),
    "sc_lambda_k_from_moments": _sig("sc_lambda_k_from_moments", c_vp, c_i32, c_i32, c_dbl, c_i32, c_i32, c_dbl,
                                     P(c_dbl), P(c_dbl)),
    "sc_normalize_rows_f32": _sig("sc_normalize_rows_f32", c_vp, c_i64, c_i32, c_vp),
    "sc_kmeans": _sig("sc_kmeans", c_vp, c_i64, c_i32, c_i32, c_i32, c_i32, c_u64, c_vp, c_vp, c_vp, P(c_dbl),
                      P(c_i32), P(c_i32), c_vp),
    "sc_ari": _sig("sc_ari", c_vp, c_vp, c_i64, P(c_dbl), c_vp),
    "sc_cluster": _sig("sc_cluster", c_vp, c_i32, c_i32, c_i32, c_i32, c_i32, c_u64, c_i32, c_i32, c_i32, c_vp, c_vp,
                       c_vp),
    "sc_stability": _sig("sc_stability", c_vp, c_i32, c_i32, c_i32, c_i32, c_i32, c_i32, c_i32, c_u64, c_i32, c_i32,
                         c_dbl, c_vp, c_vp, c_vp, c_vp, c_vp),
    "sc_nccl_unique_id": _sig("sc_nccl_unique_id", c_vp),
    "sc_comm_init": _sig("sc_comm_init", c_vp, c_i32, c_i32, P(c_vp)),
    "sc_comm_local": _sig("sc_comm_local", c_i32, c_i32, P(c_vp)),
    "sc_comm_free": _sig("sc_comm_free", c_vp),
    "sc_dist_create": _sig("sc_dist_create", c_vp, c_vp, c_i64, c_vp, c_i64, c_vp, c_vp, P(c_vp)),
    "sc_dist_free": _sig("sc_dist_free", c_vp),
    "sc_dist_filter_f32": _sig("sc_dist_filter_f32", c_vp, c_vp, c_i32, c_dbl, c_i32, c_vp, c_vp, c_vp),
    "sc_dist_lambda_max": _sig("sc_dist_lambda_max", c_vp, c_i32, c_i32, c_dbl, c_u64, c_vp, P(c_dbl), c_vp),
    "sc_dist_cheb_moments": _sig("sc_dist_cheb_moments", c_vp, c_i32, c_dbl, c_i32, c_i32, c_u64, c_vp, c_vp, c_vp),
    "sc_dist_estimate_lambda_k": _sig("sc_dist_estimate_lambda_k", c_vp, c_i32, c_i32, c_dbl, c_i32, c_i32, c_i32,
                                      c_u64, c_vp, c_i32, c_dbl, P(c_dbl), P(c_dbl), c_vp),
    "sc_dist_kmeans": _sig("sc_dist_kmeans", c_vp, c_i32, c_vp, c_vp, c_i32, c_i32, c_i32, c_i32, c_u64, c_vp, c_vp,
                           c_vp, P(c_dbl), P(c_i32), P(c_i32), c_vp),
    "sc_p2p_create": _sig("sc_p2p_create", c_vp, c_i32, c_i32, c_i64, c_vp, c_vp, c_vp, c_vp, c_i64, c_vp, c_i32,
                          P(c_vp)),
    "sc_p2p_free": _sig("sc_p2p_free", c_vp),
    "sc_p2p_export": _sig("sc_p2p_export", c_vp, c_vp),
    "sc_p2p_import": _sig("sc_p2p_import", c_vp, c_i32, c_vp),
    "sc_p2p_link_local": _sig("sc_p2p_link_local", c_vp, c_vp),
    "sc_p2p_filter_f32": _sig("sc_p2p_filter_f32", c_vp, c_vp, c_i32, c_dbl, c_i32, c_vp, c_vp, c_vp),
    "sc_p2p_filter_group_f32": _sig("sc_p2p_filter_group_f32", c_vp, c_i32, c_vp, c_i32, c_dbl, c_i32, c_vp, c_vp,
                                    c_vp),
    "sc_profile_begin": _sig("sc_profile_begin"),
    "sc_profile_end": _sig("sc_profile_end", P(c_i64), P(c_i64), P(c_dbl), P(c_dbl)),
}

EXPORTED = sorted(list(_F) + ["sc_version", "sc_last_error"])


class SCError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[sc error {code}] {msg}")
        self.code = code


def _check(rc):
    if rc != 0:
        raise SCError(rc, _lib.sc_last_error().decode(errors="replace"))


def _ptr(x):
    """Pointer of a contiguous torch tensor / numpy array (host or device), or NULL."""
    if x is None:
        return None
    if isinstance(x, np.ndarray):
        if not x.flags["C_CONTIGUOUS"]:
            raise ValueError("numpy array must be C-contiguous")
        return x.ctypes.data
    if hasattr(x, "data_ptr"):
        if not x.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return x.data_ptr()
    if isinstance(x, int):
        return x
    raise TypeError(f"cannot take the address of {type(x)}")


def _stream(stream):
    if stream is None:
        try:
            import torch
            if torch.cuda.is_available():
                return torch.cuda.current_stream().cuda_stream
        except Exception:
            pass
        return None
    if hasattr(stream, "cuda_stream"):
        return stream.cuda_stream
    return stream


def sc_version() -> int:
    return _lib.sc_version()


def sc_last_error() -> str:
    return _lib.sc_last_error().decode(errors="replace")


def sc_graph_load(n_rows, n_cols, nnz, row_ptr, col_idx, values):
    h = c_vp()
    _check(_F["sc_graph_load"](n_rows, n_cols, nnz, _ptr(row_ptr), _ptr(col_idx), _ptr(values), ctypes.byref(h)))
    return h.value


def sc_graph_free(g):
    _check(_F["sc_graph_free"](g))


def sc_graph_info(g):
    a, b, c, d = c_i64(), c_i64(), c_i64(), c_dbl()
    _check(_F["sc_graph_info"](g, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c), ctypes.byref(d)))
    return a.value, b.value, c.value, d.value


def sc_graph_strengths(g, out, stream=None):
    _check(_F["sc_graph_strengths"](g, _ptr(out), _stream(stream)))


def sc_lambda_max(g, iters=60, margin=0.01, seed=0, stream=None) -> float:
    out = c_dbl()
    _check(_F["sc_lambda_max"](g, iters, margin, seed, ctypes.byref(out), _stream(stream)))
    return out.value


def sc_cheby_coeffs(lambda_c, lambda_max, order, jackson) -> np.ndarray:
    out = np.empty(order + 1, dtype=np.float64)
    _check(_F["sc_cheby_coeffs"](lambda_c, lambda_max, order, int(jackson), out.ctypes.data))
    return out


def sc_filter_order(ratio, delta, jackson, theta=0.1, n_grid=10000, m_max=2000, stream=None):
    """-> (m_star, err); m_star 0 if no order <= m_max meets delta."""
    m = ctypes.c_int32(0)
    e = ctypes.c_double(0.0)
    _check(_F["sc_filter_order"](ratio, delta, int(jackson), theta, n_grid, m_max, ctypes.byref(m), ctypes.byref(e),
                                 _stream(stream)))
    return m.value, e.value


def sc_random_signals_f32(n, R, row0, seed, stream_id, variance, out, stream=None):
    _check(_F["sc_random_signals_f32"](n, R, row0, seed, stream_id, variance, _ptr(out), _stream(stream)))


def sc_random_signals_f64(n, R, row0, seed, stream_id, variance, out, stream=None):
    _check(_F["sc_random_signals_f64"](n, R, row0, seed, stream_id, variance, _ptr(out), _stream(stream)))


def sc_filter_apply_f32(g, coeffs, order, lambda_max, R, X, Y, stream=None):
    coeffs = np.ascontiguousarray(coeffs, dtype=np.float64)
    _check(_F["sc_filter_apply_f32"](g, coeffs.ctypes.data, order, lambda_max, R, _ptr(X), _ptr(Y), _stream(stream)))


def sc_filter_apply_f64(g, coeffs, order, lambda_max, R, X, Y, stream=None):
    coeffs = np.ascontiguousarray(coeffs, dtype=np.float64)
    _check(_F["sc_filter_apply_f64"](g, coeffs.ctypes.data, order, lambda_max, R, _ptr(X), _ptr(Y), _stream(stream)))


def sc_filter_lowpass_f32(g, lambda_c, lambda_max, order, jackson, R, seed, X, Y, stream=None):
    _check(_F["sc_filter_lowpass_f32"](g, lambda_c, lambda_max, order, int(jackson), R, seed, _ptr(X), _ptr(Y),
                                       _stream(stream)))


def sc_filter_lowpass_f64(g, lambda_c, lambda_max, order, jackson, R, seed, X, Y, stream=None):
    _check(_F["sc_filter_lowpass_f64"](g, lambda_c, lambda_max, order, int(jackson), R, seed, _ptr(X), _ptr(Y),
                                       _stream(stream)))


def sc_cheb_step_f32(g, row_begin, row_end, R, T_prev, ld_prev, T_cur, ld_cur, T_next, ld_next, Y, ld_y,
                     a, b_cur, b_prev, cy_prev, cy_cur, cy_next, y_mode, stream=None):
    _check(_F["sc_cheb_step_f32"](g, row_begin, row_end, R, _ptr(T_prev), ld_prev, _ptr(T_cur), ld_cur, _ptr(T_next),
                                  ld_next, _ptr(Y), ld_y, a, b_cur, b_prev, cy_prev, cy_cur, cy_next, y_mode,
                                  _stream(stream)))


def sc_cheb_moments(g, lambda_max, order, R, seed, X=None, stream=None) -> np.ndarray:
    mu = np.empty(2 * order + 1, dtype=np.float64)
    _check(_F["sc_cheb_moments"](g, lambda_max, order, R, seed, _ptr(X), mu.ctypes.data, _stream(stream)))
    return mu


def sc_eigencount_from_moments(moments, order, lambda_c, lambda_max, jackson) -> float:
    mu = np.ascontiguousarray(moments, dtype=np.float64)
    out = c_dbl()
    _check(_F["sc_eigencount_from_moments"](mu.ctypes.data, order, lambda_c, lambda_max, int(jackson),
                                            ctypes.byref(out)))
    return out.value


def sc_estimate_lambda_k(g, k, lambda_max, order, jackson, n_probe, seed, max_iter=40, rtol=1e-4, stream=None):
    lk, ck = c_dbl(), c_dbl()
    _check(_F["sc_estimate_lambda_k"](g, k, lambda_max, order, int(jackson), n_probe, seed, max_iter, rtol,
                                      ctypes.byref(lk), ctypes.byref(ck), _stream(stream)))
    return lk.value, ck.value


def sc_lambda_k_from_moments(moments, order, k, lambda_max, jackson, max_iter=40, rtol=1e-4):
    mu = np.ascontiguousarray(moments, dtype=np.float64)
    lk, ck = c_dbl(), c_dbl()
    _check(_F["sc_lambda_k_from_moments"](mu.ctypes.data, order, k, lambda_max, int(jackson), max_iter, rtol,
                                          ctypes.byref(lk), ctypes.byref(ck)))
    return lk.value, ck.value


def sc_normalize_rows_f32(F, n, d, stream=None):
    _check(_F["sc_normalize_rows_f32"](_ptr(F), n, d, _stream(stream)))


def sc_kmeans(F, n, d, k, restarts, max_iter, seed, uniforms, labels, centroids=None, stream=None):
    inertia, iters, best = c_dbl(), c_i32(), c_i32()
    u = None if uniforms is None else np.ascontiguousarray(uniforms, dtype=np.float64)
    _check(_F["sc_kmeans"](_ptr(F), n, d, k, restarts, max_iter, seed, _ptr(u), _ptr(labels), _ptr(centroids),
                           ctypes.byref(inertia), ctypes.byref(iters), ctypes.byref(best), _stream(stream)))
    return inertia.value, iters.value, best.value


def sc_ari(a, b, n, stream=None) -> float:
    out = c_dbl()
    _check(_F["sc_ari"](_ptr(a), _ptr(b), n, ctypes.byref(out), _stream(stream)))
    return out.value


def sc_cluster(g, k, R, order, jackson, n_probe, seed, restarts, max_iter, normalize, labels, stream=None):
    info = np.zeros(7, dtype=np.float64)
    _check(_F["sc_cluster"](g, k, R, order, int(jackson), n_probe, seed, restarts, max_iter, int(normalize),
                            _ptr(labels), info.ctypes.data, _stream(stream)))
    return info


def sc_stability(g, k_min, k_max, J, R, order, jackson, n_probe, seed, restarts, max_iter, lambda_max=0.0,
                 lambda_k=None, labels=None, stream=None):
    """-> (gamma[K], lambda_k[K]) for k = k_min..k_max; `labels` (optional) receives [K][J][n] int32."""
    K = k_max - k_min + 1
    gamma = np.empty(K, dtype=np.float64)
    lk_out = np.empty(K, dtype=np.float64)
    lk = None if lambda_k is None else np.ascontiguousarray(lambda_k, dtype=np.float64)
    _check(_F["sc_stability"](g, k_min, k_max, J, R, order, int(jackson), n_probe, seed, restarts, max_iter,
                              lambda_max, _ptr(lk), gamma.ctypes.data, lk_out.ctypes.data, _ptr(labels),
                              _stream(stream)))
    return gamma, lk_out


def sc_nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(_F["sc_nccl_unique_id"](ctypes.addressof(buf)))
    return buf.raw


def sc_comm_init(uid: bytes, world, rank):
    buf = ctypes.create_string_buffer(bytes(uid), 128)
    h = c_vp()
    _check(_F["sc_comm_init"](ctypes.addressof(buf), world, rank, ctypes.byref(h)))
    return h.value


def sc_comm_local(world, rank):
    h = c_vp()
    _check(_F["sc_comm_local"](world, rank, ctypes.byref(h)))
    return h.value


def sc_comm_free(c):
    _check(_F["sc_comm_free"](c))


def sc_dist_create(g, comm, n_interior, send_idx, send_counts, recv_counts):
    si = np.ascontiguousarray(send_idx, dtype=np.int64)
    sc_ = np.ascontiguousarray(send_counts, dtype=np.int64)
    rc = np.ascontiguousarray(recv_counts, dtype=np.int64)
    h = c_vp()
    _check(_F["sc_dist_create"](g, comm, n_interior, si.ctypes.data if si.size else None, si.size, sc_.ctypes.data,
                                rc.ctypes.data, ctypes.byref(h)))
    return h.value


def sc_dist_free(d):
    _check(_F["sc_dist_free"](d))


def sc_dist_filter_f32(d, coeffs, order, lambda_max, R, X, Y, stream=None):
    coeffs = np.ascontiguousarray(coeffs, dtype=np.float64)
    _check(_F["sc_dist_filter_f32"](d, coeffs.ctypes.data, order, lambda_max, R, _ptr(X), _ptr(Y), _stream(stream)))


def _plans(ds):
    ds = [ds] if isinstance(ds, int) else list(ds)
    arr = (c_vp * len(ds))(*ds)
    return arr, len(ds)


def _row0(row0, n):
    if row0 is None:
        return None, None
    r = np.ascontiguousarray(row0, dtype=np.int64).reshape(-1)
    assert r.size == n
    return r, r.ctypes.data


def sc_dist_lambda_max(ds, iters=60, margin=0.01, seed=0, row0=None, stream=None) -> float:
    arr, n = _plans(ds)
    keep, r0 = _row0(row0, n)
    out = c_dbl()
    _check(_F["sc_dist_lambda_max"](arr, n, iters, margin, seed, r0, ctypes.byref(out), _stream(stream)))
    return out.value


def sc_dist_cheb_moments(ds, lambda_max, order, n_probe, seed, row0=None, stream=None) -> np.ndarray:
    arr, n = _plans(ds)
    keep, r0 = _row0(row0, n)
    mu = np.zeros(2 * order + 1, dtype=np.float64)
    _check(_F["sc_dist_cheb_moments"](arr, n, lambda_max, order, n_probe, seed, r0, mu.ctypes.data, _stream(stream)))
    return mu


def sc_dist_estimate_lambda_k(ds, k, lambda_max, order, jackson, n_probe, seed, row0=None, max_iter=40, rtol=1e-4,
                              stream=None):
    arr, n = _plans(ds)
    keep, r0 = _row0(row0, n)
    lk, ck = c_dbl(), c_dbl()
    _check(_F["sc_dist_estimate_lambda_k"](arr, n, k, lambda_max, order, int(jackson), n_probe, seed, r0, max_iter,
                                           rtol, ctypes.byref(lk), ctypes.byref(ck), _stream(stream)))
    return lk.value, ck.value


def sc_dist_kmeans(comms, Fs, d, k, restarts, max_iter, seed, uniforms, labels, centroids=None, stream=None):
    """Fs / labels: per held rank, device tensors (n_local x d fp32 / n_local int32)."""
    comms = [comms] if isinstance(comms, int) else list(comms)
    n = len(comms)
    carr = (c_vp * n)(*comms)
    farr = (c_vp * n)(*[_ptr(f) for f in Fs])
    larr = (c_vp * n)(*[_ptr(x) for x in labels])
    nl = np.ascontiguousarray([int(f.shape[0]) for f in Fs], dtype=np.int64)
    u = None if uniforms is None else np.ascontiguousarray(uniforms, dtype=np.float64)
    inertia, iters, best = c_dbl(), c_i32(), c_i32()
    cp = None if centroids is None else centroids.ctypes.data
    _check(_F["sc_dist_kmeans"](carr, n, farr, nl.ctypes.data, d, k, restarts, max_iter, seed,
                                None if u is None else u.ctypes.data, larr, cp, ctypes.byref(inertia),
                                ctypes.byref(iters), ctypes.byref(best), _stream(stream)))
    return inertia.value, iters.value, best.value


def sc_p2p_create(g, world, rank, n_global, sd_ptr, sd_row, sd_peer, sd_slot, peer_n_local, max_R):
    sp = np.ascontiguousarray(sd_ptr, dtype=np.int64)
    sr = np.ascontiguousarray(sd_row, dtype=np.int64)
    pe = np.ascontiguousarray(sd_peer, dtype=np.int32)
    sl = np.ascontiguousarray(sd_slot, dtype=np.int64)
    nl = np.ascontiguousarray(peer_n_local, dtype=np.int64)
    h = c_vp()
    nd = int(sr.size)
    _check(_F["sc_p2p_create"](g, world, rank, n_global, sp.ctypes.data, sr.ctypes.data if nd else None,
                               pe.ctypes.data if nd else None, sl.ctypes.data if nd else None, nd, nl.ctypes.data,
                               max_R, ctypes.byref(h)))
    return h.value


def sc_p2p_free(p):
    _check(_F["sc_p2p_free"](p))


def sc_p2p_export(p) -> bytes:
    buf = ctypes.create_string_buffer(256)
    _check(_F["sc_p2p_export"](p, ctypes.addressof(buf)))
    return buf.raw


def sc_p2p_import(p, peer, handles: bytes):
    buf = ctypes.create_string_buffer(bytes(handles), 256)
    _check(_F["sc_p2p_import"](p, peer, ctypes.addressof(buf)))


def sc_p2p_link_local(p, peer):
    _check(_F["sc_p2p_link_local"](p, peer))


def sc_p2p_filter_f32(p, coeffs, order, lambda_max, R, X, Y, stream=None):
    coeffs = np.ascontiguousarray(coeffs, dtype=np.float64)
    _check(_F["sc_p2p_filter_f32"](p, coeffs.ctypes.data, order, lambda_max, R, _ptr(X), _ptr(Y), _stream(stream)))


def sc_p2p_filter_group_f32(ps, coeffs, order, lambda_max, R, Xs, Ys, stream=None):
    world = len(ps)
    coeffs = np.ascontiguousarray(coeffs, dtype=np.float64)
    pa = (c_vp * world)(*ps)
    xa = (c_vp * world)(*[_ptr(x) for x in Xs])
    ya = (c_vp * world)(*[_ptr(y) for y in Ys])
    _check(_F["sc_p2p_filter_group_f32"](ctypes.addressof(pa), world, coeffs.ctypes.data, order, lambda_max, R,
                                         ctypes.addressof(xa), ctypes.addressof(ya), _stream(stream)))


def sc_profile_begin():
    _check(_F["sc_profile_begin"]())


def sc_profile_end():
    """-> (launches, step_launches, step_ms, algo_bytes)"""
    a, b, c, d = c_i64(), c_i64(), c_dbl(), c_dbl()
    _check(_F["sc_profile_end"](ctypes.byref(a), ctypes.byref(b), ctypes.byref(c), ctypes.byref(d)))
    return a.value, b.value, c.value, d.value
