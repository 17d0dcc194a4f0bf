"""SVG2 (arXiv 2505.18875) sparse-attention hot path for B200 — Python binding over ``libsvg2.so``.

Argument marshalling only: every step of the path runs in the hand-written sm_100a kernels behind the C ABI
declared in ``include/svg2.h``.  PyTorch supplies device memory and the current stream.  There is no CPU or
library fallback: if the extension is missing or the device is not a B200 (sm_100), calls raise.

Names follow the ABI:
    kmeans, permute, select_topp, varblock_attention, unpermute, sparse_attention, workspace_size
and ``SVG2Attention`` keeps the per-layer centroid cache across denoising steps.
"""
from __future__ import annotations

import ctypes
import math
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SVG2_LIBRARY", os.path.join(_HERE, "libsvg2.so"))

SVG2_WARM_START = 1
SVG2_INIT_KMEANSPP = 2  # cold init by k-means++ seeding (generator DESIGN R25)
SVG2_FP8_PV = 4  # e4m3 P and V in the PV product (DESIGN R26), d = 128
(ENTRY_KMEANS, ENTRY_PERMUTE, ENTRY_SELECT_TOPP, ENTRY_VARBLOCK_ATTENTION, ENTRY_UNPERMUTE, ENTRY_SPARSE_ATTENTION,
 ENTRY_SPARSE_ATTENTION_HOST) = range(7)
STATUS = ["SVG2_OK", "SVG2_ERR_NULL_POINTER", "SVG2_ERR_INVALID_SHAPE", "SVG2_ERR_INVALID_PARAM",
          "SVG2_ERR_MISALIGNED", "SVG2_ERR_WORKSPACE_TOO_SMALL", "SVG2_ERR_UNSUPPORTED_DEVICE", "SVG2_ERR_CUDA",
          "SVG2_ERR_NOT_IMPLEMENTED"]
EXPORTED_SYMBOLS = ["svg2_status_string", "svg2_abi_version", "svg2_workspace_size", "svg2_kmeans", "svg2_permute",
                    "svg2_select_topp", "svg2_varblock_attention", "svg2_unpermute", "svg2_sparse_attention",
                    "svg2_sparse_attention_host", "svg2_sparse_attention_launch_count", "svg2_sparse_attention_ex",
                    "svg2_sparse_attention_layout"]


class SVG2Error(RuntimeError):
    def __init__(self, fn, status):
        name = STATUS[status] if 0 <= status < len(STATUS) else f"status {status}"
        super().__init__(f"{fn}: {name}")
        self.status = status


class Dims(ctypes.Structure):
    _fields_ = [("B", ctypes.c_int32), ("H", ctypes.c_int32), ("Nq", ctypes.c_int32), ("Nk", ctypes.c_int32),
                ("d", ctypes.c_int32)]


class Config(ctypes.Structure):
    _fields_ = [("Cq", ctypes.c_int32), ("Ck", ctypes.c_int32), ("iters", ctypes.c_int32), ("top_p", ctypes.c_double),
                ("scale", ctypes.c_float), ("flags", ctypes.c_uint32), ("seed", ctypes.c_uint32)]


class Debug(ctypes.Structure):
    _fields_ = [("q_labels", ctypes.c_void_p), ("k_labels", ctypes.c_void_p), ("q_perm", ctypes.c_void_p),
                ("k_perm", ctypes.c_void_p), ("q_offsets", ctypes.c_void_p), ("k_offsets", ctypes.c_void_p),
                ("mask", ctypes.c_void_p), ("events", ctypes.c_void_p * 8), ("q_objective", ctypes.c_void_p),
                ("k_objective", ctypes.c_void_p)]


class Layout(ctypes.Structure):
    _fields_ = [("q_strides", ctypes.c_int64 * 3), ("k_strides", ctypes.c_int64 * 3), ("v_strides", ctypes.c_int64 * 3),
                ("o_shards", ctypes.c_void_p), ("n_shards", ctypes.c_int32), ("shard_tokens", ctypes.c_int32),
                ("o_head_offset", ctypes.c_int32), ("part_begin", ctypes.c_int32), ("o_strides", ctypes.c_int64 * 3),
                ("part_end", ctypes.c_int32), ("part_count", ctypes.c_int32), ("aux_stream", ctypes.c_void_p),
                ("aux_events", ctypes.c_void_p * 2)]


_lib = None
_aux_cache: dict = {}


def _aux(device):
    """A high-priority stream and two events per device, lent to the fused call for its K-role fork (created once, so
    the call creates no CUDA objects of its own and keeps the role overlap under CUDA graph capture)."""
    key = device.index if device.index is not None else torch.cuda.current_device()
    got = _aux_cache.get(key)
    if got is None:
        with torch.cuda.device(key):
            st = torch.cuda.Stream(priority=-1)
            evs = [torch.cuda.Event(enable_timing=False) for _ in range(2)]
            for ev in evs:
                ev.record(st)  # materialise the handle
        got = (st, evs)
        _aux_cache[key] = got
    return got


def load_library(path: str = LIB_PATH):
    """Load libsvg2.so (raises if it was not built — there is no fallback path)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} not found: build it with `python -m paper_2505_18875_b200.build` "
                          "(or __graft_entry__.build()); the SVG2 path has no CPU fallback")
    lib = ctypes.CDLL(path)
    vp, i32, u32, sz = ctypes.c_void_p, ctypes.c_int32, ctypes.c_uint32, ctypes.c_size_t
    lib.svg2_status_string.argtypes = [ctypes.c_int]
    lib.svg2_status_string.restype = ctypes.c_char_p
    lib.svg2_abi_version.restype = ctypes.c_int
    lib.svg2_workspace_size.argtypes = [ctypes.c_int, Dims, ctypes.POINTER(Config)]
    lib.svg2_workspace_size.restype = sz
    lib.svg2_kmeans.argtypes = [vp, i32, i32, i32, i32, i32, i32, u32, u32, i32, vp, vp, vp, vp, vp, vp, vp, sz, vp]
    lib.svg2_permute.argtypes = [vp, i32, i32, i32, i32, i32, vp, vp, vp, vp, vp, vp, vp, sz, vp]
    lib.svg2_select_topp.argtypes = [vp, vp, vp, vp, i32, i32, i32, i32, i32, ctypes.c_float, ctypes.c_double, vp,
                                     vp, vp, sz, vp]
    lib.svg2_varblock_attention.argtypes = [vp, vp, vp, Dims, vp, vp, vp, i32, i32, ctypes.c_float, vp, vp, vp, vp,
                                            sz, vp]
    lib.svg2_unpermute.argtypes = [vp, vp, i32, i32, i32, i32, vp, vp]
    lib.svg2_sparse_attention.argtypes = [vp, vp, vp, Dims, ctypes.POINTER(Config), vp, vp, vp, vp,
                                          ctypes.POINTER(Debug), vp, sz, vp]
    lib.svg2_sparse_attention_ex.argtypes = [vp, vp, vp, Dims, ctypes.POINTER(Config), vp, vp, vp, vp,
                                             ctypes.POINTER(Debug), ctypes.POINTER(vp), vp, sz, vp]
    lib.svg2_sparse_attention_host.argtypes = [vp, vp, vp, Dims, ctypes.POINTER(Config), vp, vp, vp, vp, vp, sz, vp]
    lib.svg2_sparse_attention_layout.argtypes = [vp, vp, vp, Dims, ctypes.POINTER(Config), ctypes.POINTER(Layout), vp,
                                                 vp, vp, vp, ctypes.POINTER(Debug), ctypes.POINTER(vp), vp, sz, vp]
    lib.svg2_sparse_attention_launch_count.argtypes = [Dims, ctypes.POINTER(Config)]
    lib.svg2_sparse_attention_launch_count.restype = i32
    for name in ["svg2_kmeans", "svg2_permute", "svg2_select_topp", "svg2_varblock_attention", "svg2_unpermute",
                 "svg2_sparse_attention", "svg2_sparse_attention_ex", "svg2_sparse_attention_host",
                 "svg2_sparse_attention_layout"]:
        getattr(lib, name).restype = ctypes.c_int
    _lib = lib
    return lib


def _check(fn, status):
    if status != 0:
        raise SVG2Error(fn, status)


def _p(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _need(t, dtype, name, ndim=None, strided=False):
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name}: expected a CUDA tensor")
    if t.dtype != dtype:
        raise TypeError(f"{name}: expected {dtype}, got {t.dtype}")
    if strided:  # [B, H, N, d] view with d contiguous (the library takes element strides sB, sH, sN)
        if t.stride(-1) != 1:
            raise ValueError(f"{name}: the last dimension must be contiguous")
    elif not t.is_contiguous():
        raise ValueError(f"{name}: expected a contiguous tensor")
    if ndim is not None and t.dim() != ndim:
        raise ValueError(f"{name}: expected {ndim} dims, got {tuple(t.shape)}")
    return t


_ws_cache: dict = {}


def _workspace(nbytes: int, device) -> torch.Tensor:
    # one cached workspace per (device, stream): calls queued on different streams may run concurrently and must not
    # share scratch (include/svg2.h, threading)
    key = (device.index if device.index is not None else torch.cuda.current_device(),
           torch.cuda.current_stream(device).cuda_stream)
    buf = _ws_cache.get(key)
    if buf is None or buf.numel() < nbytes:
        buf = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=device)
        _ws_cache[key] = buf
    return buf


def workspace_size(entry: int, B: int, H: int, Nq: int, Nk: int, d: int, Cq: int, Ck: int = 1, iters: int = 1,
                   top_p: float = 1.0) -> int:
    lib = load_library()
    cfg = Config(Cq, Ck, iters, top_p, 0.0, 0, 0)
    return int(lib.svg2_workspace_size(entry, Dims(B, H, Nq, Nk, d), ctypes.byref(cfg)))


def _cold_flags(init: str) -> int:
    if init == "strided":
        return 0
    if init == "kmeans++":
        return SVG2_INIT_KMEANSPP
    raise ValueError(f"init must be 'strided' or 'kmeans++', not {init!r}")


def kmeans(X: torch.Tensor, C: int, iters: int, centroids: torch.Tensor | None = None, return_perm: bool = False,
           init: str = "strided", seed: int = 0, role: int = 0, return_objective: bool = False):
    """Lloyd k-means per (b,h) of X [B,H,N,d] bf16.  Warm start iff `centroids` ([B,H,C,d] f32) is given; it is
    updated in place.  Cold start: init="strided" (rows floor(jN/C), R2) or "kmeans++" with the
    generator key (seed, 2*(b*H+h) + role), role 0 = queries, 1 = keys (R25).
    Returns (labels, sizes, centroids[, perm, offsets][, objective]); objective [iters, B, H, 2] f64 =
    (J_assign, J_post) per iteration."""
    lib = load_library()
    _need(X, torch.bfloat16, "X", 4)
    B, H, N, d = X.shape
    warm = centroids is not None
    if warm:
        _need(centroids, torch.float32, "centroids", 4)
    else:
        centroids = torch.empty(B, H, C, d, dtype=torch.float32, device=X.device)
    labels = torch.empty(B, H, N, dtype=torch.int32, device=X.device)
    sizes = torch.empty(B, H, C, dtype=torch.int32, device=X.device)
    perm = torch.empty(B, H, N, dtype=torch.int32, device=X.device) if return_perm else None
    offsets = torch.empty(B, H, C + 1, dtype=torch.int32, device=X.device) if return_perm else None
    objective = torch.empty(iters, B, H, 2, dtype=torch.float64, device=X.device) if return_objective else None
    nbytes = workspace_size(ENTRY_KMEANS, B, H, N, N, d, C, iters=iters)
    ws = _workspace(max(nbytes, 256), X.device)
    flags = SVG2_WARM_START if warm else _cold_flags(init)
    _check("svg2_kmeans", lib.svg2_kmeans(_p(X), B, H, N, d, C, iters, flags, seed, role, _p(centroids),
                                          _p(labels), _p(sizes), _p(perm), _p(offsets), _p(objective), _p(ws),
                                          ws.numel(), _stream()))
    out = (labels, sizes, centroids) + ((perm, offsets) if return_perm else ()) + \
        ((objective,) if return_objective else ())
    return out


def permute(labels: torch.Tensor, C: int, X0: torch.Tensor | None = None, X1: torch.Tensor | None = None,
            d: int | None = None):
    """Stable cluster-contiguous permutation; gathers X0 / X1 ([B,H,N,d] bf16) through it.
    Returns (perm, offsets, X0p, X1p)."""
    lib = load_library()
    _need(labels, torch.int32, "labels", 3)
    B, H, N = labels.shape
    if X0 is not None:
        _need(X0, torch.bfloat16, "X0", 4)
        d = X0.shape[-1]
    if X1 is not None:
        _need(X1, torch.bfloat16, "X1", 4)
        d = X1.shape[-1]
    d = d or 128
    perm = torch.empty(B, H, N, dtype=torch.int32, device=labels.device)
    offsets = torch.empty(B, H, C + 1, dtype=torch.int32, device=labels.device)
    X0p = torch.empty_like(X0) if X0 is not None else None
    X1p = torch.empty_like(X1) if X1 is not None else None
    nbytes = workspace_size(ENTRY_PERMUTE, B, H, N, N, d, C)
    ws = _workspace(max(nbytes, 256), labels.device)
    _check("svg2_permute", lib.svg2_permute(_p(labels), B, H, N, d, C, _p(X0), _p(X0p), _p(X1), _p(X1p), _p(perm),
                                            _p(offsets), _p(ws), ws.numel(), _stream()))
    return perm, offsets, X0p, X1p


def select_topp(q_centroids, k_centroids, q_sizes, k_sizes, top_p: float, scale: float = 0.0):
    """Eq. 1 / Eq. 2 / top-p.  Returns (mask [B,H,Cq,Ck] uint8, selected_pairs [B,H] int64)."""
    lib = load_library()
    _need(q_centroids, torch.float32, "q_centroids", 4)
    _need(k_centroids, torch.float32, "k_centroids", 4)
    _need(q_sizes, torch.int32, "q_sizes", 3)
    _need(k_sizes, torch.int32, "k_sizes", 3)
    B, H, Cq, d = q_centroids.shape
    Ck = k_centroids.shape[2]
    mask = torch.empty(B, H, Cq, Ck, dtype=torch.uint8, device=q_centroids.device)
    pairs = torch.empty(B, H, dtype=torch.int64, device=q_centroids.device)
    nbytes = workspace_size(ENTRY_SELECT_TOPP, B, H, 1, 1, d, Cq, Ck)
    ws = _workspace(max(nbytes, 256), q_centroids.device)
    _check("svg2_select_topp", lib.svg2_select_topp(_p(q_centroids), _p(k_centroids), _p(q_sizes), _p(k_sizes), B, H,
                                                    Cq, Ck, d, scale, top_p, _p(mask), _p(pairs), _p(ws), ws.numel(),
                                                    _stream()))
    return mask, pairs


def varblock_attention(Qp, Kp, Vp, q_offsets, k_offsets, mask, scale: float = 0.0, q_perm=None, return_lse=False):
    """Variable-block sparse attention over permuted tensors.  With q_perm the output is in original order."""
    lib = load_library()
    for t, n in ((Qp, "Qp"), (Kp, "Kp"), (Vp, "Vp")):
        _need(t, torch.bfloat16, n, 4)
    _need(q_offsets, torch.int32, "q_offsets", 3)
    _need(k_offsets, torch.int32, "k_offsets", 3)
    _need(mask, torch.uint8, "mask", 4)
    B, H, Nq, d = Qp.shape
    Nk = Kp.shape[2]
    Cq, Ck = mask.shape[2], mask.shape[3]
    O = torch.empty_like(Qp)
    lse = torch.empty(B, H, Nq, dtype=torch.float32, device=Qp.device) if return_lse else None
    nbytes = workspace_size(ENTRY_VARBLOCK_ATTENTION, B, H, Nq, Nk, d, Cq, Ck)
    ws = _workspace(max(nbytes, 256), Qp.device)
    _check("svg2_varblock_attention",
           lib.svg2_varblock_attention(_p(Qp), _p(Kp), _p(Vp), Dims(B, H, Nq, Nk, d), _p(q_offsets), _p(k_offsets),
                                       _p(mask), Cq, Ck, scale, _p(q_perm), _p(O), _p(lse), _p(ws), ws.numel(),
                                       _stream()))
    return (O, lse) if return_lse else O


def unpermute(Op, perm):
    lib = load_library()
    _need(Op, torch.bfloat16, "Op", 4)
    _need(perm, torch.int32, "perm", 3)
    B, H, N, d = Op.shape
    O = torch.empty_like(Op)
    _check("svg2_unpermute", lib.svg2_unpermute(_p(Op), _p(perm), B, H, N, d, _p(O), _stream()))
    return O


def launch_count(B, H, Nq, Nk, d, Cq, Ck, iters, top_p, warm, init: str = "strided", fp8: bool = False) -> int:
    lib = load_library()
    flags = (SVG2_WARM_START if warm else _cold_flags(init)) | (SVG2_FP8_PV if fp8 else 0)
    cfg = Config(Cq, Ck, iters, top_p, 0.0, flags, 0)
    return int(lib.svg2_sparse_attention_launch_count(Dims(B, H, Nq, Nk, d), ctypes.byref(cfg)))


def sparse_attention(Q, K, V, Cq: int, Ck: int, iters: int, top_p: float, q_centroids=None, k_centroids=None,
                     warm: bool = False, scale: float = 0.0, debug: bool = False, events=None, out=None,
                     init: str = "strided", seed: int = 0, fp8: bool = False, input_ready=None, part=None,
                     out_shards=None):
    """The fused SVG2 call.  Q, K, V [B,H,N,d] bf16 CUDA.  q_centroids [B,H,Cq,d] / k_centroids [B,H,Ck,d] f32 are
    the centroid caches (read iff warm, always written).  Cold calls start k-means from `init` ("strided" or
    "kmeans++" with `seed`, R25).  Returns (O, selected_pairs, extras) where extras holds
    the centroids and, if debug, the intermediates (labels, perms, offsets, mask).  input_ready: None or three
    torch.cuda.Event recorded when Q, K and V are complete (svg2_sparse_attention_ex): the computation on Q starts
    while K and V are still arriving.
    Q, K, V may be strided [B,H,N,d] views with d contiguous (e.g. token-major all-to-all buffers viewed as
    [B,H,N,d]): they are read in place through svg2_sparse_attention_layout.  part = (index, count): compute only
    that part of every head's query clusters, or (begin, end, count) for parts [begin, end) (multi-GPU split,
    include/svg2.h).  out_shards = dict(shards=[tensors],
    shard_tokens=n, strides=(sB, sH, sN), head_offset=h0): write output rows straight into token-sharded buffers
    (their data pointers; peers' buffers through CUDA IPC), O is then not allocated (None is returned)."""
    lib = load_library()
    for t, n in ((Q, "Q"), (K, "K"), (V, "V")):
        _need(t, torch.bfloat16, n, 4, strided=True)
    B, H, Nq, d = Q.shape
    Nk = K.shape[2]
    dev = Q.device
    if q_centroids is None:
        if warm:
            raise ValueError("warm start needs q_centroids / k_centroids")
        q_centroids = torch.empty(B, H, Cq, d, dtype=torch.float32, device=dev)
    if k_centroids is None:
        k_centroids = torch.empty(B, H, Ck, d, dtype=torch.float32, device=dev)
    _need(q_centroids, torch.float32, "q_centroids", 4)
    _need(k_centroids, torch.float32, "k_centroids", 4)
    O = None if out_shards is not None else (out if out is not None else
                                              torch.empty(B, H, Nq, d, dtype=torch.bfloat16, device=dev))
    pairs = torch.empty(B, H, dtype=torch.int64, device=dev)
    flags = (SVG2_WARM_START if warm else _cold_flags(init)) | (SVG2_FP8_PV if fp8 else 0)
    cfg = Config(Cq, Ck, iters, top_p, scale, flags, seed)
    dims = Dims(B, H, Nq, Nk, d)
    lay = Layout()
    keep = []
    st, evs = _aux(dev)
    lay.aux_stream = st.cuda_stream
    lay.aux_events[0], lay.aux_events[1] = evs[0].cuda_event, evs[1].cuda_event
    for t, name in ((Q, "q_strides"), (K, "k_strides"), (V, "v_strides")):
        if not t.is_contiguous():
            st = [t.stride(0), t.stride(1), t.stride(2)]
            if t.shape[0] == 1:  # a size-1 dimension's stride is arbitrary in torch: any valid value
                st[0] = t.shape[1] * t.shape[2] * d
            if t.shape[1] == 1:
                st[1] = t.shape[2] * d
            getattr(lay, name)[:] = st
    if part is not None:  # (index, count) or (begin, end, count)
        part = tuple(int(x) for x in part)
        lay.part_begin, lay.part_end, lay.part_count = (part[0], part[0] + 1, part[1]) if len(part) == 2 else part
    if out_shards is not None:
        shards = out_shards["shards"]
        ptrs = (ctypes.c_void_p * len(shards))(*[int(t.data_ptr()) for t in shards])
        keep.append(ptrs)
        lay.o_shards = ctypes.cast(ptrs, ctypes.c_void_p)
        lay.n_shards = len(shards)
        lay.shard_tokens = int(out_shards["shard_tokens"])
        lay.o_strides[:] = [int(x) for x in out_shards["strides"]]
        lay.o_head_offset = int(out_shards.get("head_offset", 0))
    # 0 = invalid arguments: still call the ABI so the caller gets its precise status code
    nbytes = int(lib.svg2_workspace_size(ENTRY_SPARSE_ATTENTION, dims, ctypes.byref(cfg)))
    ws = _workspace(max(nbytes, 256), dev)
    extras = {"q_centroids": q_centroids, "k_centroids": k_centroids}
    dbg = None
    if debug or events is not None:
        dbg = Debug()
        if debug:
            extras.update(
                q_labels=torch.empty(B, H, Nq, dtype=torch.int32, device=dev),
                k_labels=torch.empty(B, H, Nk, dtype=torch.int32, device=dev),
                q_perm=torch.empty(B, H, Nq, dtype=torch.int32, device=dev),
                k_perm=torch.empty(B, H, Nk, dtype=torch.int32, device=dev),
                q_offsets=torch.empty(B, H, Cq + 1, dtype=torch.int32, device=dev),
                k_offsets=torch.empty(B, H, Ck + 1, dtype=torch.int32, device=dev),
                mask=torch.empty(B, H, Cq, Ck, dtype=torch.uint8, device=dev),
                q_objective=torch.empty(iters, B, H, 2, dtype=torch.float64, device=dev),
                k_objective=torch.empty(iters, B, H, 2, dtype=torch.float64, device=dev))
            for name in ("q_labels", "k_labels", "q_perm", "k_perm", "q_offsets", "k_offsets", "mask", "q_objective",
                         "k_objective"):
                setattr(dbg, name, extras[name].data_ptr())
        if events is not None:
            for i, ev in enumerate(events[:8]):
                if ev is None:
                    continue
                if not ev.cuda_event:  # torch creates events lazily: record once so a handle exists
                    ev.record()
                dbg.events[i] = ev.cuda_event
    ready = None
    if input_ready is not None:
        if len(input_ready) != 3:
            raise ValueError("input_ready: three events (Q, K, V)")
        ready = (ctypes.c_void_p * 3)(*[ev.cuda_event for ev in input_ready])
        if not all(ready):
            raise ValueError("input_ready: record every event before the call")
    _check("svg2_sparse_attention",
           lib.svg2_sparse_attention_layout(_p(Q), _p(K), _p(V), dims, ctypes.byref(cfg), ctypes.byref(lay),
                                            _p(q_centroids), _p(k_centroids), _p(O), _p(pairs),
                                            ctypes.byref(dbg) if dbg is not None else None,
                                            ctypes.cast(ready, ctypes.POINTER(ctypes.c_void_p)) if ready else None,
                                            _p(ws), ws.numel(), _stream()))
    return O, pairs, extras


def sparse_attention_host(Qh, Kh, Vh, Cq: int, Ck: int, iters: int, top_p: float, q_centroids=None,
                          k_centroids=None, warm: bool = False, scale: float = 0.0, out=None, init: str = "strided",
                          seed: int = 0, device=None, fp8: bool = False):
    """The fused call on HOST tensors (svg2_sparse_attention_host): Qh, Kh, Vh [B,H,N,d] bf16 CPU tensors (pin them
    for overlapped copies), output a bf16 CPU tensor (`out`, else a new pinned one).  The library streams head chunks
    to the device, computes and copies back with the transfers overlapping the computation.  Centroid caches and
    selected_pairs live on the device.  Returns (O_host, selected_pairs, extras); O_host is complete once the current
    CUDA stream has synchronised."""
    lib = load_library()
    for t, n in ((Qh, "Q"), (Kh, "K"), (Vh, "V")):
        if t.dtype != torch.bfloat16 or t.dim() != 4 or t.is_cuda or not t.is_contiguous():
            raise ValueError(f"{n}: expected a contiguous [B,H,N,d] bfloat16 CPU tensor")
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    B, H, Nq, d = Qh.shape
    Nk = Kh.shape[2]
    if q_centroids is None:
        if warm:
            raise ValueError("warm start needs q_centroids / k_centroids")
        q_centroids = torch.empty(B, H, Cq, d, dtype=torch.float32, device=dev)
    if k_centroids is None:
        k_centroids = torch.empty(B, H, Ck, d, dtype=torch.float32, device=dev)
    _need(q_centroids, torch.float32, "q_centroids", 4)
    _need(k_centroids, torch.float32, "k_centroids", 4)
    O = out if out is not None else torch.empty((B, H, Nq, d), dtype=torch.bfloat16).pin_memory()
    pairs = torch.empty(B, H, dtype=torch.int64, device=dev)
    flags = (SVG2_WARM_START if warm else _cold_flags(init)) | (SVG2_FP8_PV if fp8 else 0)
    cfg = Config(Cq, Ck, iters, top_p, scale, flags, seed)
    dims = Dims(B, H, Nq, Nk, d)
    nbytes = int(lib.svg2_workspace_size(ENTRY_SPARSE_ATTENTION_HOST, dims, ctypes.byref(cfg)))
    ws = _workspace(max(nbytes, 256), dev)
    _check("svg2_sparse_attention_host",
           lib.svg2_sparse_attention_host(_p(Qh), _p(Kh), _p(Vh), dims, ctypes.byref(cfg), _p(q_centroids),
                                          _p(k_centroids), _p(O), _p(pairs), _p(ws), ws.numel(), _stream()))
    return O, pairs, {"q_centroids": q_centroids, "k_centroids": k_centroids}


class SVG2Attention:
    """Stateful per-layer SVG2 attention with the centroid cache across denoising steps:
    the first call is a cold k-means (iters_cold), later calls warm-start from the cached centroids (iters_warm)."""

    def __init__(self, Cq: int = 100, Ck: int = 500, top_p: float = 0.9, iters_cold: int = 5, iters_warm: int = 2,
                 scale: float = 0.0):
        self.Cq, self.Ck, self.top_p = Cq, Ck, top_p
        self.iters_cold, self.iters_warm, self.scale = iters_cold, iters_warm, scale
        self.q_centroids = None
        self.k_centroids = None
        self.last_pairs = None
        self.last_nq_nk = None

    def reset(self):
        self.q_centroids = self.k_centroids = None

    def __call__(self, Q, K, V, out=None):
        B, H, N, d = Q.shape
        warm = (self.q_centroids is not None and self.q_centroids.shape == (B, H, self.Cq, d)
                and self.k_centroids.shape == (B, H, self.Ck, d))
        iters = self.iters_warm if warm else self.iters_cold
        O, pairs, ex = sparse_attention(Q, K, V, self.Cq, self.Ck, iters, self.top_p,
                                        self.q_centroids if warm else None, self.k_centroids if warm else None,
                                        warm=warm, scale=self.scale, out=out)
        self.q_centroids, self.k_centroids = ex["q_centroids"], ex["k_centroids"]
        self.last_pairs = pairs
        self.last_nq_nk = N * K.shape[2]
        return O

    def density(self) -> torch.Tensor:
        """selected pairs / (Nq Nk) per (b,h) of the last call."""
        if self.last_pairs is None:
            raise RuntimeError("density(): no call yet")
        return self.last_pairs.double() / self.last_nq_nk


def default_scale(d: int) -> float:
    """The softmax scale the library uses for scale == 0: float32(1/sqrt(d))."""
    import numpy as np
    return float(np.float32(1.0 / math.sqrt(d)))
