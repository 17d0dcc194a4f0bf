"""svg2-synth v1 — seeded synthetic Q/K/V shaped like the paper's video-DiT attention workloads.

This module is the ONLY code shared by the CUDA path's tests/bench and the oracle.  It draws random
numbers and rounds them to bf16; it contains none of the SVG2 method's arithmetic (no clustering, no
scores, no attention).  Recipe (after SURVEY.md §8(d)):

* Token grid (frames, height, width) = latent video grid, tokens in raster order (frame-major).
    tiny T = (4, 16, 16) = 1024;  Wan 480p W4 = (21, 30, 52) = 32,760;
    Wan 720p W7 = (21, 45, 80) = 75,600;  HunyuanVideo HY = (33, 45, 80) = 118,800.
* Per (b, h): numpy PCG64 seeded with 1_000_003*config_id + 1009*b + h.
  G semantic groups (64; 16 for tiny) are spatial Voronoi cells around random centres that drift per frame
  with per-group velocity ~ N(0, 0.3^2) cells/frame — objects persisting across frames, so semantically
  equal tokens are scattered in 1-D token order.  10% of tokens get a uniformly random group
  ("scattered critical tokens").
* Group directions mu_g = unit Gaussian vectors in R^d.  q_n = a*mu_g(n) + eps_n, k_n = a*mu_g(n) + eps'_n,
  eps ~ N(0, I_d);  v_n ~ N(0, I_d).  a = 8.0 (d = 128) / 6.0 (d = 64).  Everything rounded to bf16 (RNE).
* Optional 'dup' variant: 25% of tokens replaced by copies of 8 tokens (forces duplicate centroids,
  argmin ties and empty clusters).

Outputs are uint16 arrays of bf16 bit patterns, layout [B, H, N, d] contiguous.
"""
from __future__ import annotations

import dataclasses
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np


@dataclasses.dataclass(frozen=True)
class Workload:
    name: str
    config_id: int
    B: int
    H: int
    grid: tuple  # (frames, height, width)
    d: int
    Cq: int
    Ck: int
    top_p: float
    iters: int
    groups: int
    amp: float

    @property
    def N(self) -> int:
        f, h, w = self.grid
        return f * h * w


# BASELINE.json configs.  Cluster counts (100, 500) are the paper's defaults; top-p 0.9 is the
# 90%-recall operating point; iters = cold k-means iterations (warm calls use 2, R3).
WORKLOADS = {
    "tiny": Workload("tiny", 0, 1, 1, (4, 16, 16), 64, 16, 32, 0.9, 5, 16, 6.0),
    "hunyuan720p": Workload("hunyuan720p", 1, 1, 24, (33, 45, 80), 128, 100, 500, 0.9, 5, 64, 8.0),
    "wan720p": Workload("wan720p", 2, 1, 40, (21, 45, 80), 128, 100, 500, 0.9, 5, 64, 8.0),
    # HunyuanVideo calibrated to the paper's density (25.45%): a = 8.1 gives 0.258 on the
    # first warm call and ~0.25 in steady state (profiles/r02_calibration_hunyuan720p.jsonl); same seeds as above
    "hunyuan720p_r25": Workload("hunyuan720p_r25", 1, 1, 24, (33, 45, 80), 128, 100, 500, 0.9, 5, 64, 8.1),
    "wan480p": Workload("wan480p", 4, 1, 40, (21, 30, 52), 128, 100, 500, 0.9, 5, 64, 8.0),
}


def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even float32 -> bf16 bit pattern (uint16)."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    rounded = u + np.uint32(0x7FFF) + ((u >> np.uint32(16)) & np.uint32(1))
    return (rounded >> np.uint32(16)).astype(np.uint16)


def bf16_bits_to_f64(b: np.ndarray) -> np.ndarray:
    """Exact widening of bf16 bit patterns to float64."""
    return (np.asarray(b, dtype=np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32).astype(np.float64)


def _group_labels(rng, grid, G):
    T, Hh, W = grid
    centres = rng.uniform([0.0, 0.0], [Hh, W], size=(G, 2))
    vel = rng.normal(0.0, 0.3, size=(G, 2))
    yy, xx = np.meshgrid(np.arange(Hh, dtype=np.float64), np.arange(W, dtype=np.float64), indexing="ij")
    pos = np.stack([yy.ravel(), xx.ravel()], axis=1)  # [Hh*W, 2]
    labels = np.empty((T, Hh * W), np.int32)
    for t in range(T):
        c = centres + t * vel
        d2 = ((pos[:, None, :] - c[None, :, :]) ** 2).sum(-1)
        labels[t] = np.argmin(d2, axis=1)
    labels = labels.ravel()
    n = labels.shape[0]
    scatter = rng.random(n) < 0.10
    labels[scatter] = rng.integers(0, G, size=int(scatter.sum()))
    return labels


def generate_head(wl: Workload, b: int, h: int, amp: float | None = None, dup: bool = False,
                  drift_step: int = 0):
    """One (b, h) head: returns (q, k, v) uint16 bf16 bits, each [N, d].

    drift_step > 0 applies the denoising-sweep drift of SURVEY §8(d): mu_g(s) = normalise(mu_g + 0.02 s u_g)
    and AR(1) noise eps_s = 0.95 eps_{s-1} + sqrt(1 - 0.95^2) eta (config 4)."""
    a = wl.amp if amp is None else amp
    rng = np.random.Generator(np.random.PCG64(1_000_003 * wl.config_id + 1009 * b + h))
    N, d, G = wl.N, wl.d, wl.groups
    g = _group_labels(rng, wl.grid, G)
    mu = rng.standard_normal((G, d))
    mu /= np.linalg.norm(mu, axis=1, keepdims=True)
    eq = rng.standard_normal((N, d), dtype=np.float32)
    ek = rng.standard_normal((N, d), dtype=np.float32)
    v = rng.standard_normal((N, d), dtype=np.float32)
    if drift_step > 0:
        u = rng.standard_normal((G, d))
        u /= np.linalg.norm(u, axis=1, keepdims=True)
        mu = mu + 0.02 * drift_step * u
        mu /= np.linalg.norm(mu, axis=1, keepdims=True)
        rho = 0.95
        for s in range(1, drift_step + 1):
            srng = np.random.Generator(np.random.PCG64(7_777_777 + 1_000_003 * wl.config_id + 1009 * b + h + 31 * s))
            c = np.float32(np.sqrt(1.0 - rho * rho))
            eq = np.float32(rho) * eq + c * srng.standard_normal((N, d), dtype=np.float32)
            ek = np.float32(rho) * ek + c * srng.standard_normal((N, d), dtype=np.float32)
    mu32 = (a * mu).astype(np.float32)
    q = eq + mu32[g]
    k = ek + mu32[g]
    if dup:
        src = rng.integers(0, N, size=8)
        idx = rng.choice(N, size=N // 4, replace=False)
        which = src[rng.integers(0, 8, size=idx.shape[0])]
        q[idx] = q[which]
        k[idx] = k[which]
        v[idx] = v[which]
    return f32_to_bf16_bits(q), f32_to_bf16_bits(k), f32_to_bf16_bits(v)


def generate(wl: Workload, heads=None, amp: float | None = None, dup: bool = False, drift_step: int = 0,
             threads: int | None = None):
    """Full [B, H', N, d] uint16 tensors for the given head indices (default: all H heads)."""
    heads = list(range(wl.H)) if heads is None else list(heads)
    N, d = wl.N, wl.d
    q = np.empty((wl.B, len(heads), N, d), np.uint16)
    k = np.empty_like(q)
    v = np.empty_like(q)
    jobs = [(b, hi, h) for b in range(wl.B) for hi, h in enumerate(heads)]

    def run(job):
        b, hi, h = job
        q[b, hi], k[b, hi], v[b, hi] = generate_head(wl, b, h, amp=amp, dup=dup, drift_step=drift_step)

    nthreads = threads or min(len(jobs), os.cpu_count() or 1)
    if nthreads > 1:
        with ThreadPoolExecutor(nthreads) as ex:
            list(ex.map(run, jobs))
    else:
        for j in jobs:
            run(j)
    return q, k, v


def sample_rows(N: int, n: int, seed: int) -> np.ndarray:
    """Fixed-seed sample of n distinct query rows (original token order), sorted."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return np.sort(rng.choice(N, size=min(n, N), replace=False)).astype(np.int64)
