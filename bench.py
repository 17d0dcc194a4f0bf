#!/usr/bin/env python
"""bench.py — SVG2 sparse attention on B200: ms per call and effective TFLOPS vs dense, 1..8 GPUs (head-parallel).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload hunyuan720p] [--impl ours|reference]

A step = one fused svg2_sparse_attention call (k-means on Q and K warm-started from the centroid cache with 2 Lloyd
iterations, permutation, centroid top-p selection, variable-block tcgen05 attention, fused unpermute) over the whole
workload (all B*H heads; with N GPUs each rank runs H/N heads and the Ulysses all-to-all in and out).
value  = dense-equivalent effective TFLOPS = 4 N^2 d B H / t_call (whole job, max over ranks).
e2e    = the same metric through the public API with host (pinned) Q/K/V in and O out, copies inside the timing.
roofline = the variable-block attention kernel: executed algorithmic FLOPs 4 d * selected pairs / its event time,
           against the measured sustained bf16 peak (MEASURED_PEAKS.json).
cpu_baseline = the fp64 oracle (oracle/) on a bounded sample of the same workload on this host's cores.
--impl reference times that oracle as the reference arm (rank 0 only).
"""
import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "ms per sparse-attention call and effective TFLOPS at 1/2/4/8 B200 vs dense"
UNIT = "TFLOPS (dense-equivalent 4*N^2*d*B*H / t_call)"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="hunyuan720p")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--iters-warm", type=int, default=2)
    ap.add_argument("--top-p", type=float, default=None)
    ap.add_argument("--no-dense", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--fp8", action="store_true", help="e4m3 P and V in the PV product (SVG2_FP8_PV, DESIGN R26)")
    ap.add_argument("--balance", action="store_true",
                    help="N > 1: heads -> ranks by measured per-head time (dist.balanced_assignment), fixed after a "
                         "calibration step")
    ap.add_argument("--profile-once", action="store_true", help="one call only (for ncu)")
    return ap.parse_args()


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm,power.draw,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            t0 = time.time()
            while not self.lines and time.time() - t0 < 5.0:  # nvidia-smi's first sample before the timed region
                time.sleep(0.02)
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons, watts = [], 0.0, set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            try:
                watts.append(float(parts[2]))
            except ValueError:
                pass
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm.sort()
        watts.sort()
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm),
                "power_w": watts[len(watts) // 2] if watts else None}


# ----------------------------------------------------------------------------- CPU oracle baseline
def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def cpu_oracle_sample(wl, rows=4096, iters=2, heads=2):
    """The fp64 oracle as it stands on `heads` (b,h) heads of the workload: per head k-means on Q and K (cold, `iters`
    Lloyd iterations, the same work per iteration as the GPU's warm iterations), selection, and masked attention on
    `rows` sampled query rows; the per-call time is extrapolated to all rows and all B*H heads."""
    import numpy as np

    import oracle
    import svg2_synth
    oracle.build()
    scale = float(np.float32(1.0 / math.sqrt(wl.d)))
    per_head, measured, dens = [], 0.0, []
    for h in range(min(heads, wl.H)):
        q, k, v = svg2_synth.generate_head(wl, 0, h)
        Q64, K64, V64 = (svg2_synth.bf16_bits_to_f64(a) for a in (q, k, v))
        t0 = time.perf_counter()
        lq, cq, sq = oracle.kmeans(Q64, wl.Cq, iters)
        lk, ck, sk = oracle.kmeans(K64, wl.Ck, iters)
        mask, pairs = oracle.select_topp(cq, ck, sq, sk, wl.d, scale, wl.top_p)
        t1 = time.perf_counter()
        sel = svg2_synth.sample_rows(wl.N, rows, seed=h)
        oracle.attention_rows(Q64, K64, V64, scale, rows=sel, lq=lq, lk=lk, mask=mask)
        t2 = time.perf_counter()
        per_head.append((t1 - t0) + (t2 - t1) * wl.N / len(sel))
        measured += t2 - t0
        dens.append(pairs / (wl.N * wl.N))
    t_call = sum(per_head) / len(per_head) * wl.B * wl.H
    flops = 4.0 * wl.N * wl.N * wl.d * wl.B * wl.H
    return {
        "value": flops / t_call / 1e12, "unit": UNIT, "cores": os.cpu_count(), "cpu_model": cpu_model(), "kind": "oracle",
        "sample": f"{len(per_head)} of {wl.B * wl.H} heads, each: k-means Q+K ({iters} iters, full N={wl.N}), "
                  f"selection, attention on {min(rows, wl.N)} sampled rows; extrapolated to all rows and heads",
        "seconds_measured": measured, "s_per_call_extrapolated": t_call, "density": float(np.mean(dens)),
    }


def run_reference(args, wl):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    for _ in range(max(0, min(args.warmup, 1))):
        pass  # the oracle has no warm state; warm-up steps are not needed for a CPU program
    samples = [cpu_oracle_sample(wl, rows=256, heads=1) for _ in range(max(1, args.steps))]
    v = sorted(s["value"] for s in samples)[len(samples) // 2]
    t_call = sorted(s["s_per_call_extrapolated"] for s in samples)[len(samples) // 2]
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_call * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (svg2-synth v1, seeded)",
        "config": {"workload": wl.name, "B": wl.B, "H": wl.H, "N": wl.N, "d": wl.d, "Cq": wl.Cq, "Ck": wl.Ck,
                   "top_p": wl.top_p, "kmeans_iters": 2},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": os.cpu_count(), "cpu_model": cpu_model(), "kind": "oracle",
                         "sample": samples[0]["sample"] + " (one such sample per step)"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- GPU arm
def to_dev_bits(bits, dev):
    import numpy as np
    import torch
    return torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).view(torch.bfloat16).to(dev)


def dense_baseline(Q, K, V, reps=3):
    """torch SDPA on the same B200, every available backend timed; the fastest is the dense baseline."""
    import torch
    from torch.nn.attention import SDPBackend, sdpa_kernel
    res = {}
    for name, be in (("cudnn", SDPBackend.CUDNN_ATTENTION), ("flash", SDPBackend.FLASH_ATTENTION),
                     ("efficient", SDPBackend.EFFICIENT_ATTENTION)):
        try:
            with sdpa_kernel([be]):
                torch.nn.functional.scaled_dot_product_attention(Q, K, V)
                torch.cuda.synchronize()
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record()
                for _ in range(reps):
                    torch.nn.functional.scaled_dot_product_attention(Q, K, V)
                e.record()
                torch.cuda.synchronize()
                res[name] = s.elapsed_time(e) / reps
        except Exception as ex:  # backend unavailable for this shape / build
            res[name] = None
            res[name + "_error"] = str(ex).splitlines()[0][:120]
    valid = {k: v for k, v in res.items() if isinstance(v, float)}
    best = min(valid, key=valid.get) if valid else None
    return best, res


def run_ours(args, wl):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2505_18875_b200 as svg2
    import svg2_synth

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    # SVG2_BENCH_DEVICE / SVG2_DIST_BACKEND=gloo exist to exercise the multi-rank path on a single GPU (tests only);
    # a real run uses one GPU per rank and NCCL
    local_dev = int(os.environ.get("SVG2_BENCH_DEVICE", local))
    torch.cuda.set_device(local_dev)
    dev = torch.device("cuda", local_dev)
    if world > 1:
        backend = os.environ.get("SVG2_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    svg2.load_library()

    def reduce_scalar(x, op):
        """max / sum over ranks (device time is the max over ranks); CPU tensor on a CPU-only backend."""
        if world == 1:
            return x
        on = dev if dist.get_backend() == "nccl" else torch.device("cpu")
        t = torch.tensor([x], device=on, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
        return float(t.item())

    top_p = args.top_p if args.top_p is not None else wl.top_p
    from paper_2505_18875_b200.dist import (balanced_assignment, head_range, head_to_seq, heads_to_seq, seq_to_head,
                                            seq_to_head_overlapped, seq_to_heads)
    h0, h1 = head_range(wl.H, rank, world)
    Hl = h1 - h0
    # inputs: this rank's heads, full sequence (synthetic, seeded per head)
    q, k, v = svg2_synth.generate(wl, heads=range(h0, h1))
    Q, K, V = (to_dev_bits(a, dev) for a in (q, k, v))
    if world > 1:  # sequence-parallel activations as a DiT would hold them
        Qs, Ks, Vs = (head_to_seq(t) for t in (Q, K, V))
    pinned = None
    if not args.no_e2e:
        pinned = [torch.from_numpy(a.view(np.int16)).view(torch.bfloat16).pin_memory() for a in (q, k, v)]
    del q, k, v
    B, N, d = wl.B, wl.N, wl.d
    iters_w = args.iters_warm

    # cold call fills the centroid cache (the paper's first sparse step), then warm calls
    fp8 = bool(args.fp8)
    O, pairs, ex = svg2.sparse_attention(Q, K, V, wl.Cq, wl.Ck, wl.iters, top_p, fp8=fp8)
    cq, ck = ex["q_centroids"], ex["k_centroids"]
    torch.cuda.synchronize()
    assignment = None
    if args.balance and world > 1:
        # calibration: time each local head alone (warm), gather all heads' times, assign by LPT, keep it fixed
        times = []
        for hh in range(Hl):
            sl = slice(hh, hh + 1)
            Qh, Kh, Vh = (t[:, sl].contiguous() for t in (Q, K, V))
            a, b = cq[:, sl].contiguous(), ck[:, sl].contiguous()
            svg2.sparse_attention(Qh, Kh, Vh, wl.Cq, wl.Ck, iters_w, top_p, a.clone(), b.clone(), warm=True, fp8=fp8)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(2):
                svg2.sparse_attention(Qh, Kh, Vh, wl.Cq, wl.Ck, iters_w, top_p, a.clone(), b.clone(), warm=True,
                                      fp8=fp8)
            e1.record()
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1) / 2)
        on = dev if dist.get_backend() == "nccl" else torch.device("cpu")
        mine_t = torch.tensor(times, dtype=torch.float64, device=on)
        all_t = [torch.empty_like(mine_t) for _ in range(world)]
        dist.all_gather(all_t, mine_t)
        head_times = torch.cat(all_t).cpu().tolist()  # rank r holds heads [h0, h1) of the fixed split, in order
        assignment = balanced_assignment(head_times, world)
        Q, K, V = (seq_to_heads(t, assignment) for t in (Qs, Ks, Vs))
        Hl = Q.shape[1]
        if pinned is not None:
            pinned = [t.cpu().pin_memory() for t in (Q, K, V)]
        O, pairs, ex = svg2.sparse_attention(Q, K, V, wl.Cq, wl.Ck, wl.iters, top_p, fp8=fp8)  # caches of my heads
        cq, ck = ex["q_centroids"], ex["k_centroids"]
        torch.cuda.synchronize()
    if args.profile_once:
        O, pairs, _ = svg2.sparse_attention(Q, K, V, wl.Cq, wl.Ck, iters_w, top_p, cq, ck, warm=True, fp8=fp8)
        torch.cuda.synchronize()
        print(json.dumps({"profile_once": True, "density": float(pairs.double().sum()) / (B * Hl * N * N)}))
        return

    ev = [torch.cuda.Event(enable_timing=True) for _ in range(8)]

    # N > 1: Q, K, V resharded one after the other on a communication stream; the SVG2 call starts on Q while K and V
    # are in flight (svg2_sparse_attention_ex input events; env SVG2_BENCH_OVERLAP=0 reshards all three first)
    overlap = world > 1 and os.environ.get("SVG2_BENCH_OVERLAP", "1") != "0"
    comm = torch.cuda.Stream() if overlap else None

    def step(events=None):
        ready = None
        if assignment is not None:
            Qh, Kh, Vh = (seq_to_heads(t, assignment) for t in (Qs, Ks, Vs))
        elif overlap:
            (Qh, Kh, Vh), ready = seq_to_head_overlapped((Qs, Ks, Vs), comm)
        elif world > 1:
            Qh, Kh, Vh = seq_to_head(Qs), seq_to_head(Ks), seq_to_head(Vs)
        else:
            Qh, Kh, Vh = Q, K, V
        Oh, pr, _ = svg2.sparse_attention(Qh, Kh, Vh, wl.Cq, wl.Ck, iters_w, top_p, cq, ck, warm=True, events=events,
                                          fp8=fp8, input_ready=ready)
        if assignment is not None:
            return heads_to_seq(Oh, assignment, wl.H), pr
        if world > 1:
            return head_to_seq(Oh), pr
        return Oh, pr

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    stage_ms = {k_: 0.0 for k_ in ("kmeans_q", "kmeans_k", "permute", "select_topp", "worklist", "attention")}
    names = list(stage_ms)
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    per_step = []
    clocks = ClockSampler(local)
    clocks.__enter__()  # sampled through both timed loops below (the reported time is the second one)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    start.record()
    for s in range(args.steps):  # no host synchronisation inside the loop: the host enqueues ahead of the GPU
        O, pairs = step(ev)
        per_step.append(ev)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(8)]
    stop.record()
    torch.cuda.synchronize()
    for evs in per_step:
        for i, nm in enumerate(names):
            stage_ms[nm] += evs[i].elapsed_time(evs[i + 1])
    total_ms = start.elapsed_time(stop)
    t_local = total_ms / args.steps
    t_call = reduce_scalar(t_local, "max")
    if world > 1:
        dist.barrier()
    for nm in stage_ms:
        stage_ms[nm] /= args.steps
    # the loop above carries 8 stage events per call; the reported time is the plain back-to-back loop below (no events)
    start2, stop2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    start2.record()
    for _ in range(args.steps):
        step()
    stop2.record()
    torch.cuda.synchronize()
    clocks.__exit__(None, None, None)
    t_b2b_local = start2.elapsed_time(stop2) / args.steps
    t_b2b = reduce_scalar(t_b2b_local, "max")
    t_use = t_b2b
    multi = None
    if world > 1:  # SURVEY 8(e) reporting: per-rank ms, imbalance, the call without the all-to-all
        on = dev if dist.get_backend() == "nccl" else torch.device("cpu")
        mine = torch.tensor([t_b2b_local], dtype=torch.float64, device=on)
        allr = [torch.empty_like(mine) for _ in range(world)]
        dist.all_gather(allr, mine)
        per_rank = [float(t.item()) for t in allr]
        Qh, Kh, Vh = (seq_to_heads(t, assignment) for t in (Qs, Ks, Vs)) if assignment is not None else (Q, K, V)
        torch.cuda.synchronize()
        dist.barrier()
        s4, e4 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s4.record()
        for _ in range(args.steps):
            svg2.sparse_attention(Qh, Kh, Vh, wl.Cq, wl.Ck, iters_w, top_p, cq, ck, warm=True, fp8=fp8)
        e4.record()
        torch.cuda.synchronize()
        t_noa2a = reduce_scalar(s4.elapsed_time(e4) / args.steps, "max")
        multi = {"per_rank_ms": per_rank, "imbalance_max_over_mean": max(per_rank) / (sum(per_rank) / world),
                 "ms_without_all_to_all": t_noa2a, "all_to_all_share": 1.0 - t_noa2a / t_b2b if t_b2b > 0 else None,
                 "heads_per_rank": Hl}

    pairs_local = float(pairs.double().sum().item())
    pairs_total = reduce_scalar(pairs_local, "sum")
    density = pairs_total / (B * wl.H * N * N)
    dense_flops = 4.0 * N * N * d * B * wl.H
    value = dense_flops / (t_use * 1e-3) / 1e12
    pk, pk_src = peaks()
    attn_ms = stage_ms["attention"]
    attn_flops_local = 4.0 * d * pairs_local
    achieved = attn_flops_local / (attn_ms * 1e-3) / 1e12
    # FP8 PV: half the algorithmic FLOPs (PV) run at the e4m3 rate = 2 x bf16 (the guide's nominal ratio applied to
    # the measured bf16 peak), so the peak of the mix is the harmonic mean over the two equal halves, 4/3 x bf16
    peak = pk["bf16_tflops_sustained"] * (4.0 / 3.0 if fp8 else 1.0)
    roofline = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                "frac": achieved / peak, "traffic": None,
                "kernel": "k_varblock_attn<128> (tcgen05 QK^T + PV, fused unpermute)" + (", e4m3 PV" if fp8 else ""),
                "peak_source": f"{pk_src} bf16 sustained (cuBLAS 8192^3 back-to-back, MEASURED_PEAKS.json)"
                + (" for QK^T, x2 (nominal fp8/bf16) for PV, harmonic mix" if fp8 else ""),
                "algorithmic": "4*d*selected_pairs executed FLOPs per launch / event time of the launch"}
    traffic_file = os.path.join(ROOT, "profiles", f"traffic_{wl.name}{'_fp8' if fp8 else ''}.json")
    if os.path.exists(traffic_file):
        try:
            roofline["traffic"] = json.load(open(traffic_file)).get("dram_bytes_per_launch")
        except Exception:
            pass

    # ---- e2e through the C-ABI call on HOST buffers (svg2_sparse_attention_host, rank-local heads): every step moves
    # this rank's Q, K, V from pinned host memory to the device and O back, inside the library's pipeline
    e2e = None
    if pinned is not None and world > 1 and assignment is None:
        # N > 1: what a sequence-parallel caller does per step -- its token shard of Q, K, V [B, N/P, H, d] from pinned
        # host memory to the device, the Ulysses reshard in (overlapped with the k-means, input-ready events), the
        # fused call on this rank's heads, the reshard out, and its O shard back to pinned host memory
        hs = [t.cpu().pin_memory() for t in (Qs, Ks, Vs)]
        ds = [torch.empty_like(t) for t in (Qs, Ks, Vs)]
        o_host = torch.empty(tuple(Qs.shape), dtype=torch.bfloat16).pin_memory()
        qc_e, kc_e = cq.clone(), ck.clone()
        comm_e = torch.cuda.Stream()

        def e2e_step():
            for dd, hh in zip(ds, hs):
                dd.copy_(hh, non_blocking=True)
            (Qh, Kh, Vh), ready = seq_to_head_overlapped(tuple(ds), comm_e)
            Oh, _, _ = svg2.sparse_attention(Qh, Kh, Vh, wl.Cq, wl.Ck, iters_w, top_p, qc_e, kc_e, warm=True, fp8=fp8,
                                             input_ready=ready)
            o_host.copy_(head_to_seq(Oh), non_blocking=True)

        e2e_step()
        torch.cuda.synchronize()
        dist.barrier()
        s3, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s3.record()
        for _ in range(args.steps):
            e2e_step()
        e3.record()
        torch.cuda.synchronize()
        te = reduce_scalar(s3.elapsed_time(e3) / args.steps, "max")
        nbytes = int(reduce_scalar(float(Qs.numel() * 2), "sum"))
        e2e = {"value": dense_flops / (te * 1e-3) / 1e12, "unit": UNIT, "ms_per_step": te,
               "h2d_bytes_per_step": 3 * nbytes, "d2h_bytes_per_step": nbytes,
               "api": "token shards from pinned host -> Ulysses all-to-all (dist.seq_to_head_overlapped) -> "
                      "sparse_attention -> all-to-all back -> pinned host"}
    elif pinned is not None:
        out_host = torch.empty((B, Hl, N, d), dtype=torch.bfloat16).pin_memory()
        qc_e, kc_e = cq.clone(), ck.clone()

        def e2e_step():
            svg2.sparse_attention_host(pinned[0], pinned[1], pinned[2], wl.Cq, wl.Ck, iters_w, top_p, qc_e, kc_e,
                                       warm=True, out=out_host, fp8=fp8)

        e2e_step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        s3, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s3.record()
        for _ in range(args.steps):
            e2e_step()
        e3.record()
        torch.cuda.synchronize()
        te = s3.elapsed_time(e3) / args.steps
        te = reduce_scalar(te, "max")
        nbytes = int(reduce_scalar(float(B * Hl * N * d * 2), "sum"))  # all ranks (uneven with --balance)
        e2e = {"value": dense_flops / (te * 1e-3) / 1e12, "unit": UNIT, "ms_per_step": te,
               "h2d_bytes_per_step": 3 * nbytes, "d2h_bytes_per_step": nbytes,
               "api": "svg2_sparse_attention_host (C ABI, pinned host Q/K/V in, host O out)"}

    # ---- dense baseline (same box, same inputs)
    dense = None
    if not args.no_dense and rank == 0:
        best, res = dense_baseline(Q, K, V)
        if best:
            t_dense = res[best] * wl.H / Hl  # this rank's heads on one GPU; scale to all heads on one GPU
            dense = {"best_backend": best, "ms_per_call_1gpu_all_heads": t_dense, "backends_ms_rank_heads": res,
                     "speedup_vs_dense": t_dense / (t_use * world) if world == 1 else None,
                     "inv_density": 1.0 / density if density > 0 else None,
                     "kernel_speedup_vs_dense": (res[best] / attn_ms) if attn_ms > 0 else None,
                     "paper_bar_0.85_over_density": 0.85 / density if density > 0 else None}
    # ---- tile-work multiplier: MMA area the kernel executes / algorithmic area, from one debug call
    # outside the timed region (this rank's heads): Q tiles of 128 rows per query cluster; key stream = runs of
    # adjacent selected key clusters, each padded to whole 8-row groups, the stream rounded up to 16 keys (DESIGN 6)
    _, _, dx = svg2.sparse_attention(Q, K, V, wl.Cq, wl.Ck, iters_w, top_p, cq.clone(), ck.clone(), warm=True,
                                     debug=True, fp8=fp8)
    q_off = dx["q_offsets"].cpu().numpy().astype(np.int64).reshape(-1, wl.Cq + 1)
    k_off = dx["k_offsets"].cpu().numpy().astype(np.int64).reshape(-1, wl.Ck + 1)
    msk = dx["mask"].cpu().numpy().astype(bool).reshape(-1, wl.Cq, wl.Ck)
    alg = exe = 0
    for hh in range(msk.shape[0]):
        sq, sk = np.diff(q_off[hh]), np.diff(k_off[hh])
        alg += int((sq * (msk[hh] @ sk)).sum())
        for i in range(wl.Cq):
            m = msk[hh, i] & (sk > 0)
            run = np.cumsum(m & ~np.concatenate(([False], m[:-1]))) * m  # run id per selected cluster, 0 = none
            run_len = np.bincount(run, weights=sk * m)[1:]
            stream = np.ceil(np.ceil(run_len / 8).sum() * 8 / 16) * 16
            exe += int(np.ceil(sq[i] / 128) * 128 * stream)
    tile_work = exe / alg if alg else None
    cpu = None
    if not args.no_cpu and rank == 0 and world == 1:
        cpu = cpu_oracle_sample(wl, rows=4096, iters=iters_w, heads=2)
    launches = svg2.launch_count(B, Hl, N, N, d, wl.Cq, wl.Ck, iters_w, top_p, True, fp8=fp8) * args.steps
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_use, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "bf16 + e4m3 PV" if fp8 else "bf16",
            "data": "synthetic (svg2-synth v1: seeded Voronoi-group Q/K/V, bf16, shapes of the named workload)",
            "config": {"workload": wl.name, "B": B, "H": wl.H, "N": N, "d": d, "Cq": wl.Cq, "Ck": wl.Ck,
                       "top_p": top_p, "kmeans_iters": iters_w, "warm_start": True, "pv": "e4m3" if fp8 else "bf16",
                       "parallelism": f"head-parallel x{world}" + (" + Ulysses all-to-all" if world > 1 else "")
                       + (" (heads balanced by measured time)" if assignment is not None else ""),
                       "l2": "inputs larger than L2 (Q+K+V = %.2f GB > 126 MB)" % (3 * B * wl.H * N * d * 2 / 1e9)},
            "density": density, "ms_per_call": t_use, "ms_per_call_with_stage_events": t_call,
            "stages_ms": stage_ms, "gpu_launches": launches, "roofline": roofline, "e2e": e2e,
            "dense_baseline": dense, "cpu_baseline": cpu, "clocks": clocks.summary(),
            "attention_executed_tflops": achieved, "tile_work_multiplier": tile_work,
            "head_assignment": assignment, "multi_gpu": multi,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    args = parse()
    import svg2_synth
    wl = svg2_synth.WORKLOADS[args.workload]
    if args.impl == "reference":
        run_reference(args, wl)
    else:
        run_ours(args, wl)


if __name__ == "__main__":
    main()
