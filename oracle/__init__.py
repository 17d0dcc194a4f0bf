"""fp64 CPU oracle for the SVG2 hot path (arXiv 2505.18875) — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference``) may import this package.  It shares no code with the CUDA product path
(``paper_2505_18875_b200``) and neither imports the other; the only common dependency is the
seeded input generator ``svg2_synth``, which holds none of the method's arithmetic.

The arithmetic lives in ``svg2_oracle.c`` (plain C, fp64, OpenMP over independent rows), each
function citing the PAPER.md passage it follows.  This module only marshals numpy arrays.

Per-(b,h) functions:
    kmeans(X, C, iters, init=None)            PAPER.md:259, 322-326   (Lloyd, strided cold init R2)
    identification.*                          recall / density / miss / waste / PSNR / position blocks (8(f) row 3)
    assign(X, centroids)                      one assign step + best/second distances (R16 tie bands)
    permute(labels, C)                        PAPER.md:275            (stable counting sort)
    select_topp(cq, ck, sq, sk, d, scale, p)  PAPER.md:296-315        (Eq. 1, Eq. 2, top-p)
    attention_rows(Q, K, V, ..., rows)        PAPER.md:194-197, 329-334 (masked, renormalised)
    dense_rows(Q, K, V, scale, rows)
    sparse_attention_head(...)                the whole per-head pipeline, composed from the above
Parity status: see DESIGN.md §Oracle (k-means on realistic data beyond invariants: "parity unpinned").
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "svg2_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")
_vp = ctypes.c_void_p


def build(force: bool = False) -> str:
    """Compile liboracle.so (gcc, fp64, no fast-math, no FP contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(
            ["gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
             "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is not None:
        return _lib
    build()
    lib = ctypes.CDLL(_LIB)
    i64, i32, dbl = ctypes.c_int64, ctypes.c_int, ctypes.c_double
    lib.oracle_kmeans.argtypes = [_dp, i64, i32, i32, i32, _vp, _i32p, _dp, _i64p, _vp, _vp]
    lib.oracle_kmeans.restype = i32
    lib.oracle_assign.argtypes = [_dp, i64, i32, i32, _dp, _i32p, _vp, _vp]
    lib.oracle_assign.restype = None
    lib.oracle_permute.argtypes = [_i32p, i64, i32, _i32p, _i64p]
    lib.oracle_permute.restype = i32
    lib.oracle_select_topp.argtypes = [_dp, _dp, _i64p, _i64p, i32, i32, i32, dbl, dbl, _u8p,
                                       ctypes.POINTER(i64), _vp, _vp, _vp]
    lib.oracle_select_topp.restype = i32
    lib.oracle_attention_rows.argtypes = [_dp, _dp, _dp, i64, i64, i32, _vp, _vp, _vp, i32, dbl,
                                          _vp, i64, _dp, _vp]
    lib.oracle_attention_rows.restype = i32
    u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
    lib.oracle_philox4x32_10.argtypes = [u32p, u32p, u32p]
    lib.oracle_philox4x32_10.restype = None
    lib.oracle_kmeanspp_init.argtypes = [_dp, i64, i32, i32, ctypes.c_uint32, ctypes.c_uint32, _i64p]
    lib.oracle_kmeanspp_init.restype = i32
    _lib = lib
    return lib


def _ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def kmeans(X, C, iters, init=None, return_objective=False):
    """Lloyd k-means on one (b,h) role.  X [N,d].  Returns labels int32 [N], centroids f64 [C,d],
    sizes int64 [C] (and J_assign, J_post [iters] if requested)."""
    lib = _load()
    X = _f64(X)
    N, d = X.shape
    labels = np.empty(N, np.int32)
    cent = np.empty((C, d), np.float64)
    sizes = np.empty(C, np.int64)
    ja = np.empty(iters, np.float64)
    jp = np.empty(iters, np.float64)
    init_a = None if init is None else _f64(init).reshape(C, d)
    rc = lib.oracle_kmeans(X, N, d, C, iters, _ptr(init_a), labels, cent, sizes, _ptr(ja), _ptr(jp))
    if rc != 0:
        raise ValueError(f"oracle_kmeans: invalid arguments (N={N}, C={C}, iters={iters})")
    if return_objective:
        return labels, cent, sizes, ja, jp
    return labels, cent, sizes


def philox4x32_10(ctr, key):
    """The counter-based generator of DESIGN R25: 4 x uint32 out for a 4 x uint32 counter and 2 x uint32 key."""
    out = np.empty(4, np.uint32)
    _load().oracle_philox4x32_10(np.asarray(ctr, np.uint32), np.asarray(key, np.uint32), out)
    return out


def kmeanspp_stream(b, h, H, role):
    """R25 stream id of one (b, h) and role (0 = Q, 1 = K)."""
    return 2 * (b * H + h) + role


def kmeanspp_init(X, C, seed, stream):
    """k-means++ cold start (generator R25): the C picked row indices, int64 [C]."""
    X = _f64(X)
    N, d = X.shape
    idx = np.empty(C, np.int64)
    rc = _load().oracle_kmeanspp_init(X, N, d, C, seed, stream, idx)
    if rc != 0:
        raise ValueError(f"oracle_kmeanspp_init: invalid arguments (N={N}, C={C})")
    return idx


def kmeanspp(X, C, iters, seed, stream, return_objective=False):
    """Cold k-means with the k-means++ init: Lloyd iterations from the picked rows.  Returns labels, centroids,
    sizes (and J_assign, J_post) like kmeans(), plus the picked indices."""
    X = _f64(X)
    idx = kmeanspp_init(X, C, seed, stream)
    res = kmeans(X, C, iters, init=X[idx], return_objective=return_objective)
    return (*res, idx)


def assign(X, centroids):
    """One assign step: labels, best distance d1, second-best distance d2 (exact fp64)."""
    lib = _load()
    X = _f64(X)
    cent = _f64(centroids)
    N, d = X.shape
    C = cent.shape[0]
    labels = np.empty(N, np.int32)
    d1 = np.empty(N, np.float64)
    d2 = np.empty(N, np.float64)
    lib.oracle_assign(X, N, d, C, cent, labels, _ptr(d1), _ptr(d2))
    return labels, d1, d2


def permute(labels, C):
    """Stable cluster-contiguous permutation: perm int32 [N] (pos -> original), offsets int64 [C+1]."""
    lib = _load()
    labels = np.ascontiguousarray(labels, dtype=np.int32)
    N = labels.shape[0]
    perm = np.empty(N, np.int32)
    offsets = np.empty(C + 1, np.int64)
    if lib.oracle_permute(labels, N, C, perm, offsets) != 0:
        raise ValueError("oracle_permute: label out of range")
    return perm, offsets


def select_topp(cq, ck, sq, sk, d, scale, p, return_tables=False):
    """Eq. 1/2 + top-p.  Returns mask uint8 [Cq,Ck], selected_pairs int (and S, W, Z if requested)."""
    lib = _load()
    cq = _f64(cq)
    ck = _f64(ck)
    sq = np.ascontiguousarray(sq, dtype=np.int64)
    sk = np.ascontiguousarray(sk, dtype=np.int64)
    Cq, Ck = cq.shape[0], ck.shape[0]
    mask = np.empty((Cq, Ck), np.uint8)
    pairs = ctypes.c_int64(0)
    S = np.empty((Cq, Ck), np.float64) if return_tables else None
    W = np.empty((Cq, Ck), np.float64) if return_tables else None
    Z = np.empty(Cq, np.float64) if return_tables else None
    rc = lib.oracle_select_topp(cq, ck, sq, sk, Cq, Ck, d, float(scale), float(p), mask,
                                ctypes.byref(pairs), _ptr(S), _ptr(W), _ptr(Z))
    if rc != 0:
        raise ValueError(f"oracle_select_topp: top_p must be in (0, 1], got {p}")
    if return_tables:
        return mask, pairs.value, S, W, Z
    return mask, pairs.value


def attention_rows(Q, K, V, scale, rows=None, lq=None, lk=None, mask=None, return_lse=False):
    """Masked (or dense, if mask is None) attention for the given query rows (original order)."""
    lib = _load()
    Q, K, V = _f64(Q), _f64(K), _f64(V)
    Nq, d = Q.shape
    Nk = K.shape[0]
    if rows is None:
        rows_a = None
        nrows = Nq
    else:
        rows_a = np.ascontiguousarray(rows, dtype=np.int64)
        nrows = rows_a.shape[0]
    O = np.empty((nrows, d), np.float64)
    lse = np.empty(nrows, np.float64)
    if mask is not None:
        lq = np.ascontiguousarray(lq, dtype=np.int32)
        lk = np.ascontiguousarray(lk, dtype=np.int32)
        mask = np.ascontiguousarray(mask, dtype=np.uint8)
        Ck = mask.shape[1]
    else:
        Ck = 0
    rc = lib.oracle_attention_rows(Q, K, V, Nq, Nk, d, _ptr(lq), _ptr(lk), _ptr(mask), Ck, float(scale),
                                   _ptr(rows_a), nrows, O, _ptr(lse))
    if rc != 0:
        raise ValueError("oracle_attention_rows: a query row has an empty key set (contract violation)")
    return (O, lse) if return_lse else O


def dense_rows(Q, K, V, scale, rows=None):
    return attention_rows(Q, K, V, scale, rows=rows)


def sparse_attention_head(Q, K, V, Cq, Ck, iters, top_p, scale=None, init_q=None, init_k=None, rows=None):
    """The whole SVG2 pipeline for one (b,h), in original token order (no permutation).
    Returns dict(O, labels_q, labels_k, cent_q, cent_k, sizes_q, sizes_k, mask, pairs)."""
    Q, K, V = _f64(Q), _f64(K), _f64(V)
    d = Q.shape[1]
    if scale is None:
        scale = 1.0 / np.sqrt(d)
    lq, cq, sq = kmeans(Q, Cq, iters, init=init_q)
    lk, ck, sk = kmeans(K, Ck, iters, init=init_k)
    mask, pairs = select_topp(cq, ck, sq, sk, d, scale, top_p)
    O = attention_rows(Q, K, V, scale, rows=rows, lq=lq, lk=lk, mask=mask)
    return dict(O=O, labels_q=lq, labels_k=lk, cent_q=cq, cent_k=ck, sizes_q=sq, sizes_k=sk,
                mask=mask, pairs=pairs)


def flops_from_pairs(pairs, d):
    """Sparse attention FLOPs = 4 d * selected token pairs (QK^T and PV multiply-adds)."""
    return 4 * int(d) * int(pairs)
