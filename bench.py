#!/usr/bin/env python
"""bench.py -- decode-step attention latency and effective HBM GB/s of the S^2ANTA hot path
(BASELINE.json metric) on B200.

Default (N=1): BASELINE config 2 -- Llama-3.1-8B GQA decode (H=32, H_kv=8, d=128, bf16),
32k context, batch 1, S=256 stratified, synthetic W1 (i.i.d. Gaussian) inputs.  Under
torchrun with N ranks every rank runs its own config-2 problem with global batch id = rank
(batch x kv-head sharding, no data-path collective -> weak scaling); NCCL is used only for
the barrier and the max-over-ranks of the device times.  Extra legs at N > 1: config 3 as stated
(32 sequences sharded over the N GPUs, strong scaling) and config 4 (one 512k sequence sharded
over the N GPUs, sharding.seqshard_decode with its NCCL all-gather and all-reduce timed inside).

Timing (headline): W untimed warm-up steps, then K back-to-back steps bracketed by barrier +
synchronize and CUDA events on the launching stream; the steps rotate over >= 4 distinct KV caches
(512 MiB, > 4x the 126 MB L2), so every step streams its K from HBM -- the "inputs larger than L2"
option (no flush between the timed steps).  isolated_latency_us is the other protocol: one call
between CUDA events after a 512 MiB L2-flush write (the paper's).

value = algorithmic bytes of all ranks / max-over-ranks mean step time, where algorithmic
bytes = all K bytes + UNIQUE sampled V rows (union over the GQA group) + q + out
(SURVEY sec. 8(d)).  `--impl reference` times the fp64 CPU oracle (the reference arm of
this tier) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "decode-step attention µs and effective HBM GB/s (% of B200 peak) at 32k ctx"
WORKLOAD = ("BASELINE config 2: Llama-3.1-8B GQA decode (32 q / 8 kv heads, d=128, bf16), 32k context, "
            "batch 1 per GPU, S=256 stratified")
PAPER_CONTEXT = ("paper (RTX 6000 Ada, sm_89): S2ANTA-prop S=128 1.50x and S2ANTA-flash S=2048 1.51x "
                 "decode-kernel speedup over FlashInfer at 32k (PAPER.md:212); no absolute us published")
REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
           0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
           0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=400)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--batch", type=int, default=1, help="sequences per GPU")
    ap.add_argument("--seqlen", type=int, default=32768)
    ap.add_argument("--S", type=int, default=256)
    ap.add_argument("--mode", default="stratified", choices=["iid", "stratified", "systematic"])
    ap.add_argument("--workload", default="gauss", choices=["gauss", "temp4", "sink"])
    ap.add_argument("--page-size", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip dense/graph/e2e/profiled legs")
    ap.add_argument("--seed", type=int, default=0x5A17A)
    ap.add_argument("--no-baselines", action="store_true", help="skip the FlashInfer / FA-2 / SDPA context timings")
    ap.add_argument("--no-config3", action="store_true", help="skip the BASELINE config-3 (batch 32) S sweep")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="process-group backend for N > 1 (gloo + --share-gpu: exercise the multi-rank legs "
                         "on one GPU; never a bench number)")
    ap.add_argument("--share-gpu", action="store_true", help="every rank on cuda:0 (test mode, with gloo)")
    ap.add_argument("--config", type=int, default=2, choices=[1, 2, 3, 4, 5],
                    help="BASELINE config whose leg to print alone (2 = the default headline line)")
    return ap.parse_args()


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy read+write)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def load_traffic(path="two_kernel"):
    """dram bytes per launch of the dominant kernel of `path` from the committed ncu --set full
    summaries (profiles/dominant_kernel_ncu.json, config 2)."""
    p = os.path.join(ROOT, "profiles", "dominant_kernel_ncu.json")
    if os.path.exists(p):
        try:
            d = json.load(open(p))
            return d.get(path, {}).get("dram_bytes_per_launch")
        except Exception:
            return None
    return None


class ClockSampler:
    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,power.draw")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # nvidia-smi's NVML start-up (tens of ms) must not overlap the ~1 ms timed loop: wait for
            # its first sample; it keeps sampling every 50 ms through the timed region
            t0 = time.time()
            while not self.rows and time.time() - t0 < 3.0:
                time.sleep(0.005)
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 3:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            self.proc.wait(timeout=5)
            self.t.join(timeout=2)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        reasons = set()
        for r in self.rows:
            try:
                bits = int(r[2], 16)
            except ValueError:
                continue
            for b, n in REASONS.items():
                if bits & b and n != "gpu_idle":
                    reasons.add(n)
        busy = sorted(sm)[len(sm) // 2:] if sm else []
        return {"sm_mhz": statistics.median(busy) if busy else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


def algorithmic_bytes(seqlens, Hkv, d, e, uniq_rows, B, H):
    """K bytes (all keys) + unique sampled V rows + q + out."""
    kb = sum(seqlens) * Hkv * d * e
    vb = uniq_rows * d * e
    return kb, vb, 2 * B * H * d * e


def run_reference(args, rank, world):
    """Reference arm of this tier: the fp64 CPU oracle, as it stands, on a bounded sample of
    the workload (2 of the 8 kv-head groups of the config-2 step per timed step)."""
    import numpy as np
    from threadpoolctl import threadpool_info

    import santa_inputs as si
    from oracle import santa_oracle as o

    if rank != 0:
        return None
    H, Hkv, d, n = 32, 8, 128, args.seqlen
    inp = si.make_decode_inputs(1, H, Hkv, d, n, dtype="bf16", workload=args.workload, seed=0)
    groups = 2
    q = si.as_bits(inp.q)[:, :4 * groups]
    K = si.as_bits(inp.K)[:, :groups]
    V = si.as_bits(inp.V)[:, :groups]
    times, uniq = [], []
    for step in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        out, idx = o.santa_decode(q, K, V, [n], args.S, args.mode, args.seed, step)
        dt = time.perf_counter() - t0
        if step >= args.warmup:
            times.append(dt)
            uniq.append(sum(o.unique_rows(idx[0, 4 * g:4 * g + 4]) for g in range(groups)))
    e = 2
    kb, vb, qo = algorithmic_bytes([n], groups, d, e, float(np.mean(uniq)), 1, 4 * groups)
    t = float(np.mean(times))
    cores = max([x.get("num_threads", 1) for x in threadpool_info()] + [1])
    value = (kb + vb + qo) / t / 1e9
    sample = f"config-2 step restricted to {groups} of 8 kv-head groups ({4 * groups} q heads), fp64 oracle"
    return {
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(t * 1e3, 3),
        "us_per_step": round(t * 1e6, 1), "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded torch.randn, W1 Gaussian)",
        "config": {"workload": WORKLOAD, "sample": sample, "S": args.S, "mode": args.mode},
        "cpu_baseline": {"value": round(value, 4), "unit": "GB/s", "cores": cores, "kind": "oracle",
                         "sample": sample, "threads": {"python_loop": 1, "blas": cores},
                         "cpu_model": cpu_model(), "nproc": os.cpu_count()},
        "e2e": {"value": round(value, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def cpu_baseline(inp_cpu, args, bytes_per_step):
    """The oracle as it stands (fp64 numpy; a Python loop over (b, h) whose only multi-threaded
    step is the BLAS mat-vec of the scores) timed on this host on the full config-2 step: once with
    BLAS limited to one thread and once with all cores (~5 s each), plus BASELINE config 1 (one
    head, 1024 keys, d = 64, fp32, S = 16 systematic) in seconds."""
    import numpy as np
    from threadpoolctl import threadpool_info, threadpool_limits

    import santa_inputs as si
    from oracle import santa_oracle as o

    q, K, V = si.as_bits(inp_cpu.q), si.as_bits(inp_cpu.K), si.as_bits(inp_cpu.V)
    sl = inp_cpu.seqlens.cpu().numpy()

    def run(budget):
        times = []
        t_start = time.perf_counter()
        while time.perf_counter() - t_start < budget or len(times) < 2:
            t0 = time.perf_counter()
            o.santa_decode(q, K, V, sl, args.S, args.mode, args.seed, len(times))
            times.append(time.perf_counter() - t0)
        return float(np.median(times)), len(times), time.perf_counter() - t_start

    with threadpool_limits(limits=1):
        t1, n1, w1 = run(5.0)
    t_all, n_all, w_all = run(5.0)
    blas = max([x.get("num_threads", 1) for x in threadpool_info()] + [1])
    c1 = si.make_decode_inputs(1, 1, 1, 64, 1024, dtype="f32", seed=1)
    c1t = []
    for i in range(7):
        t0 = time.perf_counter()
        o.santa_decode(si.as_bits(c1.q), si.as_bits(c1.K), si.as_bits(c1.V), [1024], 16, "systematic", args.seed, i)
        c1t.append(time.perf_counter() - t0)
    return {"value": round(bytes_per_step / t_all / 1e9, 4), "unit": "GB/s", "cores": blas, "kind": "oracle",
            "sample": f"full config-2 step (batch {inp_cpu.q.shape[0]}), {n_all} steps in {w_all:.1f} s, "
                      f"median {t_all * 1e3:.0f} ms/step",
            "threads": {"python_loop": 1, "blas": blas}, "cpu_model": cpu_model(), "nproc": os.cpu_count(),
            "single_thread": {"value": round(bytes_per_step / t1 / 1e9, 4), "unit": "GB/s",
                              "ms_per_step": round(t1 * 1e3, 1), "steps": n1},
            "all_cores": {"value": round(bytes_per_step / t_all / 1e9, 4), "unit": "GB/s",
                          "ms_per_step": round(t_all * 1e3, 1), "steps": n_all},
            "config1_seconds": round(float(np.median(c1t)), 5),
            "language": "numpy fp64 (the oracle as committed, not the C++ program SURVEY 8(c) sketched)"}


def library_baselines(probs, NR, timed_loop, args):
    """The paper's comparison systems (FlashInfer decode, FlashAttention-2 decode) and torch SDPA
    on the same caches and protocol -- context for the paper's 1.5x claim, not a target.
    Library kernels; a failure is reported, never fatal."""
    import torch

    res = {}
    Ks = [p.K.transpose(1, 2).contiguous() for p in probs]   # sequence-major [B, n, Hkv, d]
    Vs = [p.V.transpose(1, 2).contiguous() for p in probs]
    for i in range(args.warmup):
        pass
    try:
        from flash_attn import flash_attn_with_kvcache
        sl = probs[0].seqlens
        fn = lambda i: flash_attn_with_kvcache(probs[i % NR].q.unsqueeze(1), Ks[i % NR], Vs[i % NR],  # noqa: E731
                                               cache_seqlens=sl)
        for i in range(args.warmup):
            fn(i)
        res["flash_attn_2_decode_us"] = round(timed_loop(fn, args.steps) * 1e3, 2)
    except Exception as e:  # noqa: BLE001
        res["flash_attn_2_decode_us"] = f"unavailable: {type(e).__name__}: {str(e)[:120]}"
    try:
        import flashinfer
        fn = lambda i: flashinfer.single_decode_with_kv_cache(probs[i % NR].q[0], Ks[i % NR][0], Vs[i % NR][0])  # noqa: E731
        for i in range(args.warmup):
            fn(i)
        res["flashinfer_decode_us"] = round(timed_loop(fn, args.steps) * 1e3, 2)
    except Exception as e:  # noqa: BLE001
        res["flashinfer_decode_us"] = f"unavailable: {type(e).__name__}: {str(e)[:120]}"
    try:
        fn = lambda i: torch.nn.functional.scaled_dot_product_attention(  # noqa: E731
            probs[i % NR].q.unsqueeze(2), probs[i % NR].K, probs[i % NR].V, enable_gqa=True)
        for i in range(args.warmup):
            fn(i)
        res["torch_sdpa_us"] = round(timed_loop(fn, args.steps) * 1e3, 2)
    except Exception as e:  # noqa: BLE001
        res["torch_sdpa_us"] = f"unavailable: {type(e).__name__}: {str(e)[:120]}"
    res["note"] = "same caches, back-to-back protocol; dense exact attention (reads 2x the KV bytes)"
    return res


def unique_rows_gpu(idx, Hkv):
    """Distinct sampled V rows per (b, kv-head), summed (GQA dedup: the G heads of a group share V)."""
    import torch
    B, H, S = idx.shape
    g = idx.reshape(B, Hkv, (H // Hkv) * S).sort(dim=-1).values
    return int(B * Hkv + (g[..., 1:] != g[..., :-1]).sum().item())


def config3(args, dev, stream, timed_loop, max_over_ranks, peak, world):
    """BASELINE config 3: batch 32 per GPU, 32k, S in {64,128,256,512} stratified -- the same
    decode step on a 4 GiB KV cache (> L2: back-to-back steps stream from HBM), plus the in-repo
    dense decode on the same cache.  value-style GB/s = algorithmic bytes / step time."""
    import torch

    import paper_2605_01910_b200 as santa
    import santa_inputs as si

    B, H, Hkv, d, n = 32, 32, 8, 128, args.seqlen
    inp = si.make_decode_inputs(B, H, Hkv, d, n, dtype="bf16", workload=args.workload, seed=77, device=str(dev))
    geo = santa.make_geometry(inp.q, Hkv, n, batch_offset=int(os.environ.get("RANK", "0")) * B)
    out = torch.empty_like(inp.q)
    steps = max(3, min(args.steps, 10))
    rows = {}
    kb = B * Hkv * n * d * 2
    for S in (64, 128, 256, 512):
        ws = santa.workspace(geo, S, dev)
        idx = torch.empty((B, H, S), dtype=torch.int32, device=dev)
        santa.santa_decode_attention(geo, inp.q, inp.K, inp.V, inp.seqlens, S, args.mode, args.seed, 0, out, idx,
                                     ws, stream)
        torch.cuda.synchronize()
        U = unique_rows_gpu(idx, Hkv)
        fn = lambda i: santa.santa_decode_attention(geo, inp.q, inp.K, inp.V, inp.seqlens, S, args.mode,  # noqa
                                                    args.seed, i, out, None, ws, stream)
        for i in range(3):
            fn(i)
        t = max_over_ranks(timed_loop(fn, steps))
        byt = kb + U * d * 2 + 2 * B * H * d * 2
        gb = byt / (t * 1e-3) / 1e9
        rows[str(S)] = {"us": round(t * 1e3, 2), "GBps": round(gb, 1), "frac_of_peak": round(gb / peak, 4),
                        "unique_rows": U}
    dws = santa.workspace(geo, 1, dev)
    fn = lambda i: santa.santa_dense_reference(geo, inp.q, inp.K, inp.V, inp.seqlens, out, dws, stream)  # noqa
    for i in range(2):
        fn(i)
    t = max_over_ranks(timed_loop(fn, steps))
    rows["dense_reference"] = {"us": round(t * 1e3, 2), "GBps": round(2 * kb / (t * 1e-3) / 1e9, 1)}
    rows["note"] = ("BASELINE config 3 per GPU: batch 32, 32k, stratified; one KV cache of 4 GiB (> L2), "
                    f"{steps} back-to-back steps; {world} GPU(s), batch x kv-head sharding (weak scaling)")
    del inp, out
    torch.cuda.empty_cache()
    return rows


def config4(args, dev, stream, timed_loop, peak):
    """BASELINE config 4 on ONE GPU: 512k context, S=1024 stratified, the per-rank work of a
    sequence-sharded step for R = 2/4/8 ranks (rank 0's shard of 512k/R tokens): phase 1 (score
    pass + shard (m_r, L_r)) and phase 2 (global shard CDF, own strata, local gather).  The NCCL
    all_gather / all_reduce between them are not timed here (one GPU in this run); the stats of the
    other ranks are taken equal to this rank's (each rank owns ~S/R strata), labelled as such."""
    import torch

    from paper_2605_01910_b200 import sharding
    import santa_inputs as si

    H, Hkv, d, S, n = 32, 8, 128, 1024, 524288
    rows = {}
    for R in (2, 4, 8):
        nloc = n // R
        inp = si.make_decode_inputs(1, H, Hkv, d, nloc, dtype="bf16", workload=args.workload, seed=400 + R,
                                    device=str(dev))
        be = sharding.CudaBackend()
        st = be.stats(inp.q, inp.K, inp.seqlens, Hkv, S)
        stats_all = st.unsqueeze(0).repeat(R, 1, 1, 1).contiguous()
        off = torch.zeros(1, dtype=torch.int32, device=dev)
        steps = max(3, min(args.steps, 20))
        t1 = timed_loop(lambda i: be.stats(inp.q, inp.K, inp.seqlens, Hkv, S), steps)
        t2 = timed_loop(lambda i: be.sample_gather(stats_all, 0, R, off, inp.V, inp.seqlens, S, args.mode, args.seed,
                                                   i), steps)
        kb = Hkv * nloc * d * 2
        rows[str(R)] = {"tokens_per_rank": nloc, "phase1_us": round(t1 * 1e3, 2), "phase2_us": round(t2 * 1e3, 2),
                        "per_rank_kernel_us": round((t1 + t2) * 1e3, 2),
                        "phase1_GBps": round(kb / (t1 * 1e-3) / 1e9, 1),
                        "phase1_frac_of_peak": round(kb / (t1 * 1e-3) / 1e9 / peak, 4)}
        del inp, be, st, stats_all
        torch.cuda.empty_cache()
    rows["note"] = ("per-rank kernels only (1 GPU): rank 0 of R, shard = 512k/R tokens of every kv head, "
                    "S=1024; the two NCCL collectives (all_gather of R x 256 B, all_reduce of 16 KiB) are "
                    "exercised by the gloo tests, not timed here")
    return rows


def config1(args, dev, stream, timed_loop, peak):
    """BASELINE config 1: one head, n_k = 1024, d = 64, fp32, S = 16 systematic, batch 1 -- launch-bound
    (its purpose is the CPU oracle in seconds and fp32 parity); no roofline claim."""
    import torch

    import paper_2605_01910_b200 as santa
    import santa_inputs as si

    inp = si.make_decode_inputs(1, 1, 1, 64, 1024, dtype="f32", seed=1, device=str(dev))
    geo = santa.make_geometry(inp.q, 1, 1024)
    ws = santa.workspace(geo, 16, dev)
    out = torch.empty_like(inp.q)
    fn = lambda i: santa.santa_decode_attention(geo, inp.q, inp.K, inp.V, inp.seqlens, 16, "systematic",  # noqa
                                                args.seed, i, out, None, ws, stream)
    for i in range(10):
        fn(i)
    t = timed_loop(fn, max(10, min(args.steps, 200)))
    return {"us": round(t * 1e3, 2), "path": santa.santa_auto_path(geo, 16),
            "note": "1 head x 1024 keys x d=64 fp32, S=16 systematic: launch-bound, no roofline claim"}


def config5(args, dev, stream, timed_loop, peak):
    """BASELINE config 5: Bernoulli ternary-q score stage (mean-group, stratified, B=8) + the
    S^2ANTA value stage (S=256 stratified), 32k context, batch 16, feature-major K^T; calibrated
    lognormal queries.  Bytes = the selected feature rows of K^T + unique V rows."""
    import torch

    import paper_2605_01910_b200 as santa
    import santa_inputs as si

    Bt, H, Hkv, d, n, S, nB = 16, 32, 8, 128, args.seqlen, 256, 8
    inp = si.make_decode_inputs(Bt, H, Hkv, d, n, dtype="bf16", workload="lognormal", seed=500,
                                feature_major=True, device=str(dev))
    inp.K = None  # only the feature-major copy is read
    torch.cuda.empty_cache()
    geo = santa.make_geometry(inp.q, Hkv, n)
    ws = santa.workspace(geo, S, dev)
    out = torch.empty_like(inp.q)
    idx = torch.empty((Bt, H, S), dtype=torch.int32, device=dev)
    scores = torch.empty((Bt, H, n), dtype=torch.float32, device=dev)
    mask = torch.zeros((Bt, Hkv, d), dtype=torch.uint8, device=dev)
    santa.santa_bernoulli_scores(geo, inp.q, inp.Kt, inp.seqlens, nB, 1, 1, args.seed, 0, scores, mask, ws)
    santa.santa_decode_attention_bernoulli(geo, inp.q, inp.Kt, inp.V, inp.seqlens, nB, 1, 1, S, args.mode, args.seed,
                                           0, out, idx, ws)
    torch.cuda.synchronize()
    frac = float(mask.float().mean().item())
    U = unique_rows_gpu(idx, Hkv)
    fn = lambda i: santa.santa_decode_attention_bernoulli(geo, inp.q, inp.Kt, inp.V, inp.seqlens, nB, 1, 1, S,  # noqa
                                                          args.mode, args.seed, i, out, None, ws, stream)
    for i in range(3):
        fn(i)
    steps = max(3, min(args.steps, 20))
    t = timed_loop(fn, steps)
    byt = frac * Bt * Hkv * d * n * 2 + U * d * 2 + 2 * Bt * H * d * 2
    gb = byt / (t * 1e-3) / 1e9
    del inp, out, scores, ws
    torch.cuda.empty_cache()
    return {"us": round(t * 1e3, 2), "GBps": round(gb, 1), "frac_of_peak": round(gb / peak, 4),
            "feature_access_frac": round(frac, 4), "unique_rows": U,
            "note": "batch 16, 32k, mean-group stratified Bernoulli B=8 (P:448, P:510) + S=256 stratified; "
                    "bytes = selected K^T feature rows + unique V rows + q/out"}


def config3_strong(args, dev, stream, timed_loop, max_over_ranks, peak, world, rank):
    """BASELINE config 3 as stated -- 32 sequences of 32k SHARDED over the N GPUs by (batch, kv-head)
    units (sharding.plan_units: contiguous slabs, global Philox ids, no collective): each rank holds
    and decodes only its slabs; step time = max over ranks; GB/s = all 32 sequences' algorithmic
    bytes / that time (strong scaling: total work fixed)."""
    import torch

    import paper_2605_01910_b200 as santa
    from paper_2605_01910_b200 import sharding
    import santa_inputs as si

    B, H, Hkv, d, n = 32, 32, 8, 128, args.seqlen
    G = H // Hkv
    slabs = sharding.plan_units(B, Hkv, world)[rank]
    parts = []
    for sl in slabs:
        nb, nk = sl.b1 - sl.b0, sl.k1 - sl.k0
        inp = si.make_decode_inputs(nb, nk * G, nk, d, n, dtype="bf16", workload=args.workload,
                                    seed=7700 + sl.b0 * Hkv + sl.k0, device=str(dev))
        geo = santa.make_geometry(inp.q, nk, n, batch_offset=sl.b0, head_offset=sl.k0 * G)
        parts.append((inp, geo, torch.empty_like(inp.q)))
    steps = max(3, min(args.steps, 10))
    rows = {}
    for S in (64, 128, 256, 512):
        wss = [santa.workspace(geo, S, dev) for _, geo, _ in parts]

        def fn(i, S=S, wss=wss):
            for (inp, geo, out), ws in zip(parts, wss):
                santa.santa_decode_attention(geo, inp.q, inp.K, inp.V, inp.seqlens, S, args.mode, args.seed, i, out,
                                             None, ws, stream)
        for i in range(3):
            fn(i)
        t = max_over_ranks(timed_loop(fn, steps))
        # unique V rows are counted on rank-local slabs and summed over ranks (bytes of the whole job)
        U = 0
        for (inp, geo, out), ws in zip(parts, wss):
            idx = torch.empty((inp.q.shape[0], inp.q.shape[1], S), dtype=torch.int32, device=dev)
            santa.santa_decode_attention(geo, inp.q, inp.K, inp.V, inp.seqlens, S, args.mode, args.seed, 0, out, idx,
                                         ws, stream)
            U += unique_rows_gpu(idx, geo.n_kv_heads)
        U = sum_over_ranks(float(U), dev, world)
        byt = B * Hkv * n * d * 2 + U * d * 2 + 2 * B * H * d * 2
        rows[str(S)] = {"us": round(t * 1e3, 2), "GBps": round(byt / (t * 1e-3) / 1e9, 1),
                        "per_gpu_frac_of_peak": round(byt / world / (t * 1e-3) / 1e9 / peak, 4)}
        del wss
    rows["note"] = (f"32 sequences x 32k sharded over {world} GPU(s) by (batch, kv-head) units "
                    f"({sum(s.units for s in slabs)} units on rank {rank}); max over ranks; strong scaling")
    del parts
    torch.cuda.empty_cache()
    return rows


def sum_over_ranks(x, dev, world):
    import torch
    import torch.distributed as dist
    if world == 1:
        return x
    t = torch.tensor([x], device=dev, dtype=torch.float64)
    dist.all_reduce(t)
    return float(t.item())


def config4_seqshard(args, dev, stream, timed_loop, max_over_ranks, peak, world, rank):
    """BASELINE config 4 on N GPUs: one 512k-token sequence, S = 1024 stratified by shard mass, each
    rank holding the contiguous 512k / N tokens of every kv head; sharding.seqshard_decode with the
    CUDA backend -- phase 1 (score pass + shard (m_r, L_r)), the all-gather of the [1, 32, 2] fp64
    stats over the process group, phase 2 (global shard CDF, own strata, local gather), the
    all-reduce of the [1, 32, 128] fp32 partial outputs -- timed end to end with both collectives
    inside the events (max over ranks), and the two kernel phases alone."""
    import torch

    from paper_2605_01910_b200 import sharding
    import santa_inputs as si

    H, Hkv, d, S, n = 32, 8, 128, 1024, 524288
    seqlens = torch.tensor([n], dtype=torch.int32, device=dev)
    ranges = sharding.shard_ranges([n], rank, world, dev)
    nloc = int(ranges[1][0].item())
    loc = si.make_decode_inputs(1, H, Hkv, d, nloc, dtype="bf16", workload=args.workload, seed=900 + rank,
                                device=str(dev))
    q = si.make_decode_inputs(1, H, Hkv, d, 16, dtype="bf16", seed=899, device=str(dev)).q  # same q everywhere
    be = sharding.CudaBackend()
    steps = max(3, min(args.steps, 20))

    def full(i):
        sharding.seqshard_decode(q, loc.K, loc.V, seqlens, S, args.mode, args.seed, i, backend=be, ranges=ranges)
    for i in range(3):
        full(i)
    t = max_over_ranks(timed_loop(full, steps))
    st = be.stats(q, loc.K, ranges[1], Hkv, S)
    stats_all = st.unsqueeze(0).repeat(world, 1, 1, 1).contiguous()
    t1 = max_over_ranks(timed_loop(lambda i: be.stats(q, loc.K, ranges[1], Hkv, S), steps))
    t2 = max_over_ranks(timed_loop(lambda i: be.sample_gather(stats_all, rank, world, ranges[0], loc.V, ranges[1], S,
                                                              args.mode, args.seed, i), steps))
    kb = Hkv * n * d * 2
    out = {"R": world, "us": round(t * 1e3, 2), "GBps": round(kb / (t * 1e-3) / 1e9, 1),
           "per_gpu_frac_of_peak": round(kb / world / (t * 1e-3) / 1e9 / peak, 4),
           "kernel_only_us": {"phase1": round(t1 * 1e3, 2), "phase2": round(t2 * 1e3, 2)},
           "collectives_us": round(max(0.0, t - t1 - t2) * 1e3, 2),
           "note": ("seqshard_decode end to end (score pass, all_gather of (m_r, L_r), sampler + gather, "
                    f"all_reduce of the partials) over {args.dist_backend}; GB/s counts the K bytes of the "
                    "whole 512k sequence")}
    if not args.share_gpu:
        # the same step with both exchanges as one-shot peer-memory kernels (CUDA-IPC mapped buffers,
        # NVLink P2P stores + flags); never with ranks sharing one GPU (they would wait on each other).
        # Every rank must agree on whether the mapping worked before any rank launches a peer kernel.
        ex, err = None, ""
        try:  # all ranks raise together if any rank cannot map the buffers (PeerExchange)
            ex = sharding.PeerExchange(1 * H * d * 4, device=dev)
        except Exception as e:  # e.g. no P2P / IPC between the GPUs of this node
            err = repr(e)[:200]
        if ex is not None:
            def full_peer(i):
                sharding.seqshard_decode(q, loc.K, loc.V, seqlens, S, args.mode, args.seed, i, backend=be,
                                         ranges=ranges, exchange=ex)
            for i in range(3):
                full_peer(i)
            tp = max_over_ranks(timed_loop(full_peer, steps))
            out["peer_exchange"] = {"us": round(tp * 1e3, 2), "GBps": round(kb / (tp * 1e-3) / 1e9, 1),
                                    "collectives_us": round(max(0.0, tp - t1 - t2) * 1e3, 2),
                                    "note": "santa_peer_allgather + santa_peer_allreduce_f32 instead of NCCL"}
            ex.close()
        else:
            out["peer_exchange"] = {"unavailable": err}
    del loc, be
    torch.cuda.empty_cache()
    return out


def peer_exchange_emulated(args, dev, timed_loop):
    """The two config-4 exchange kernels on ONE GPU with every rank emulated in one cooperative launch
    (local buffers, no NVLink): the kernels' own cost beside the NCCL-free path's latency budget."""
    import torch

    from paper_2605_01910_b200 import sharding
    rows = {}
    K = 20
    for R in (2, 4, 8):
        grp = sharding.EmulatedPeerGroup(R, 32 * 128 * 4, device=dev)
        st = [torch.randn(1, 32, 2, dtype=torch.float64, device=dev) for _ in range(R)]
        pt = [torch.randn(1, 32, 128, device=dev) for _ in range(R)]
        res = {}
        for name, fn in (("allgather_512B_us", lambda: grp.all_gather(st)), ("allreduce_16KiB_us",
                                                                            lambda: grp.all_reduce_(pt))):
            fn()
            torch.cuda.synchronize()
            # K calls (epochs e+1 .. e+K, each its own kernel parameters) captured in one CUDA graph:
            # the device time per exchange without the Python / ctypes launch path in the way
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                for _ in range(K):
                    fn()
            g.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            res[name] = round(e0.elapsed_time(e1) / K * 1e3, 2)
        rows[str(R)] = res
    rows["note"] = ("all R ranks of the group in ONE cooperative launch on one GPU (EmulatedPeerGroup), 20 calls "
                    "replayed from a CUDA graph: device time per exchange without NVLink (local buffers); a "
                    "multi-GPU rank (n_local = 1, plain launch) adds the P2P store latency")
    return rows


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        res = run_reference(args, rank, world)
        if res is not None:
            print(json.dumps(res), flush=True)
        return

    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2605_01910_b200 as santa
    import santa_inputs as si

    dev = torch.device("cuda", 0 if args.share_gpu else local)
    torch.cuda.set_device(dev)
    if world > 1:
        if args.dist_backend == "nccl":
            os.environ["NCCL_DEBUG"] = "INFO"            # comm_nranks / nvls / channels on stderr
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT,TUNING")
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")

    B, H, Hkv, d, n = args.batch, 32, 8, 128, args.seqlen
    G = H // Hkv
    stream = torch.cuda.current_stream()
    prob_bytes = 2 * B * Hkv * n * d * 2
    NR = max(1, -(-(512 << 20) // prob_bytes))  # rotate >= 512 MiB (> 4x L2) of distinct KV caches

    class Prob:
        pass

    probs = []
    for r in range(NR):
        inp = si.make_decode_inputs(B, H, Hkv, d, n, dtype="bf16", workload=args.workload,
                                    seed=1000 * rank + r, page_size=args.page_size, device=str(dev))
        p = Prob()
        p.inp = inp
        p.q = inp.q
        if args.page_size:
            p.K, p.V, p.pt = inp.K_pool, inp.V_pool, inp.page_table
        else:
            p.K, p.V, p.pt = inp.K, inp.V, None
        p.seqlens = inp.seqlens
        # every rank owns global batch ids rank*B .. rank*B+B-1 (batch x kv-head sharding)
        p.geo = santa.make_geometry(p.q, Hkv, n, p.pt, args.page_size, batch_offset=rank * B)
        p.out = torch.empty_like(p.q)
        probs.append(p)
    ws = santa.workspace(probs[0].geo, args.S, dev)
    idx = torch.empty((B, H, args.S), dtype=torch.int32, device=dev)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def step(i, with_idx=False):
        p = probs[i % NR]
        santa.santa_decode_attention(p.geo, p.q, p.K, p.V, p.seqlens, args.S, args.mode, args.seed, i, p.out,
                                     idx if with_idx else None, ws, stream)

    # unique V rows per step (algorithmic V bytes), measured on offsets 0..3 outside timing
    uniq = []
    for i in range(4):
        step(i, True)
        torch.cuda.synchronize()
        ii = idx.cpu().numpy()
        uniq.append(sum(len(np.unique(ii[b, g * G:(g + 1) * G])) for b in range(B) for g in range(Hkv)))
    U = float(np.mean(uniq))
    kb, vb, qo = algorithmic_bytes([n] * B, Hkv, d, 2, U, B, H)
    bytes_step = kb + vb + qo

    def timed_loop(fn, K):
        """K back-to-back calls bracketed by barrier + synchronize; device time per call (ms)."""
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        for i in range(K):
            fn(i)
        e1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        return e0.elapsed_time(e1) / K

    def local_loop(fn, K):
        """timed_loop without the cross-rank barriers: for legs one rank runs alone (rank 0's library
        baselines), where a barrier would pair with another rank's unrelated collective."""
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        for i in range(K):
            fn(i)
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / K

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    if args.config != 2:  # one BASELINE config's leg alone, as its own JSON line
        peak, peak_src = load_peaks()
        legs = {1: lambda: config1(args, dev, stream, timed_loop, peak),
                3: lambda: config3(args, dev, stream, timed_loop, max_over_ranks, peak, world),
                4: lambda: (config4(args, dev, stream, timed_loop, peak) if world == 1 else
                            config4_seqshard(args, dev, stream, timed_loop, max_over_ranks, peak, world, rank)),
                5: lambda: config5(args, dev, stream, timed_loop, peak)}
        with ClockSampler(local) as clk:
            leg = legs[args.config]()
        if rank == 0:
            print(json.dumps({"metric": METRIC, "config": {"baseline_config": args.config}, "n_gpus": world,
                              "result": leg, "peak_GBps": peak, "peak_source": peak_src, "clocks": clk.summary()}),
                  flush=True)
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return
    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        ms = max_over_ranks(timed_loop(lambda i: step(args.warmup + i), args.steps))
        t_end = time.time() + 1.0  # keep the same workload running ~1 s for the clock sampler
        j = 0
        while time.time() < t_end:
            for _ in range(50):
                step(j)
                j += 1
            torch.cuda.synchronize()
    value = world * bytes_step / (ms * 1e-3) / 1e9

    peak, peak_src = load_peaks()
    res = {
        "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms, 5), "us_per_step": round(ms * 1e3, 2),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (seeded torch.randn, W1 i.i.d. Gaussian, PAPER.md:1757-1760)",
        "config": {"workload": WORKLOAD, "batch_per_gpu": B, "seq_len": n, "S": args.S, "mode": args.mode,
                   "n_heads": H, "n_kv_heads": Hkv, "head_dim": d, "page_size": args.page_size or "contiguous",
                   "inputs": args.workload,
                   "l2": f"inputs larger than L2: {NR} distinct KV caches ({NR * prob_bytes >> 20} MiB) rotated "
                         f"across back-to-back steps; isolated_latency_us uses a 512 MiB L2-flush write instead",
                   "parallelism": f"batch x kv-head sharding over {world} GPU(s), no data-path collective"},
        "bytes_per_step": {"K": kb, "V_unique": vb, "q_out": qo, "unique_rows": U,
                           "V_per_sample_convention": B * H * args.S * d * 2},
        "pct_of_peak": {"measured_copy": round(100 * value / world / peak, 1),
                        "spec_8TBps": round(100 * value / world / 8000.0, 1)},
        "clocks": clk.summary(),
        # score pass + sampler kernel per step on the two-kernel path, one launch on the step kernels
        "gpu_launches": args.steps * (2 if santa.santa_auto_path(probs[0].geo, args.S) == "two_kernel" else 1),
        "paper_context": PAPER_CONTEXT,
    }

    auto = santa.santa_auto_path(probs[0].geo, args.S)  # the path santa_decode_attention takes
    res["path"] = auto
    if not args.no_extras:
        # the score pass alone (the streaming half of the two-kernel path), back-to-back
        def score(i):
            p = probs[i % NR]
            santa.santa_score_phase(p.geo, p.q, p.K, p.seqlens, ws, stream)
        for i in range(args.warmup):
            score(i)
        sms = max_over_ranks(timed_loop(score, args.steps))
        p0 = probs[0]
        santa.santa_score_phase(p0.geo, p0.q, p0.K, p0.seqlens, ws, stream)

        def sample(i):
            santa.santa_sample_phase(p0.geo, p0.V, p0.seqlens, args.S, args.mode, args.seed, i, p0.out, None, ws,
                                     stream)
        sgms = max_over_ranks(timed_loop(sample, args.steps))
        sach = (kb + B * H * d * 2) / (sms * 1e-3) / 1e9
        # (1) the dominant kernel of the AUTO path: the score pass (two-kernel path) or the step
        # kernel itself (one launch per step); CUDA events on the launching stream
        if auto == "two_kernel":
            res["roofline"] = {"bound": "hbm", "achieved": round(sach, 1), "peak": peak, "unit": "GB/s",
                               "frac": round(sach / peak, 4), "traffic": load_traffic(auto),
                               "kernel": "score_stream_kernel<bf16,128,4,5,2> (split-KV score pass, interleaved)",
                               "peak_source": peak_src, "algorithmic_bytes_per_launch": kb + B * H * d * 2,
                               "kernel_us": round(sms * 1e3, 2),
                               "timing": ("the pass alone, back-to-back over rotating KV caches > 4x L2, CUDA events; "
                                          "launches PDL-chained (each waits for its predecessor before touching memory, "
                                          "its launch and set-up overlap the predecessor's tail; a serialised cold "
                                          "launch under ncu is ~17 us)"),
                               "sample_phase_us": round(sgms * 1e3, 2), "share_of_step": round(sms / ms, 3)}
        else:
            achieved = bytes_step / (ms * 1e-3) / 1e9
            res["roofline"] = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                               "frac": round(achieved / peak, 4), "traffic": load_traffic(auto),
                               "kernel": f"santa_{auto}_kernel (whole step in one launch)", "peak_source": peak_src,
                               "algorithmic_bytes_per_launch": bytes_step, "kernel_us": round(ms * 1e3, 2),
                               "timing": "back-to-back launches over rotating KV caches > 4x L2, CUDA events",
                               "share_of_step": 1.0}
        # (1b) every execution path on the same protocol
        paths = {}
        for pth in ("two_kernel", "step", "step_tc"):
            def stepp(i, pth=pth):
                p = probs[i % NR]
                santa.santa_decode_attention_path(p.geo, p.q, p.K, p.V, p.seqlens, args.S, args.mode, args.seed, i,
                                                  p.out, None, ws, pth, stream)
            try:
                for i in range(args.warmup):
                    stepp(i)
                t = max_over_ranks(timed_loop(stepp, args.steps))
                paths[pth] = {"us_per_step": round(t * 1e3, 2), "GBps": round(bytes_step / (t * 1e-3) / 1e9, 1)}
            except Exception as ex:  # noqa: BLE001 -- a path not eligible for this geometry
                paths[pth] = f"unavailable: {ex}"[:120]
        paths["score_phase"] = {"kernel": "score_stream_kernel<bf16,128,4,5,2>", "us": round(sms * 1e3, 2),
                                "achieved_GBps": round(sach, 1), "frac": round(sach / peak, 4)}
        paths["sample_phase_us"] = round(sgms * 1e3, 2)
        res["paths"] = paths
        # (1c) S^2ANTA-prop (the paper's own estimator): score pass + budget/count/gather
        # kernel, at this S and at the paper's prop operating point S = 128
        prop = {"estimator": "S^2ANTA-prop, largest-remainder tile budgets, B_tile = 64 (App. M)"}
        for Sp in sorted({args.S, 128}):
            pws = santa.workspace(p0.geo, Sp, dev)
            pidx = torch.empty((B, H, Sp), dtype=torch.int32, device=dev)
            pu = []
            for i in range(4):
                santa.santa_decode_attention_prop(p0.geo, p0.q, p0.K, p0.V, p0.seqlens, Sp, args.seed, i, p0.out,
                                                  pidx, pws, stream)
                torch.cuda.synchronize()
                ii = pidx.cpu().numpy()
                pu.append(sum(len(np.unique(ii[b, g * G:(g + 1) * G])) for b in range(B) for g in range(Hkv)))
            pkb, pvb, pqo = algorithmic_bytes([n] * B, Hkv, d, 2, float(np.mean(pu)), B, H)

            def propp(i, Sp=Sp, pws=pws):
                p = probs[i % NR]
                santa.santa_decode_attention_prop(p.geo, p.q, p.K, p.V, p.seqlens, Sp, args.seed, i, p.out, None,
                                                  pws, stream)
            for i in range(args.warmup):
                propp(i)
            t = max_over_ranks(timed_loop(propp, args.steps))
            prop[f"S{Sp}"] = {"us_per_step": round(t * 1e3, 2),
                              "GBps": round((pkb + pvb + pqo) / (t * 1e-3) / 1e9, 1),
                              "frac": round((pkb + pvb + pqo) / (t * 1e-3) / 1e9 / peak, 4),
                              "unique_rows": float(np.mean(pu)), "launches_per_step": 2}
            del pws
        res["prop"] = prop
        # (1d) S^2ANTA-flash at the paper's operating point (tile 256, S = 2048)
        # and at this S: score pass + per-tile draw / merge-weighted gather kernel
        flash = {"estimator": "S^2ANTA-flash, uniform per-tile budgets + LSE merge (App. N)"}
        for Sf, tile in ((2048, 256), (args.S, 256)):
            fws = santa.workspace(p0.geo, Sf, dev)
            Mf = santa.santa_flash_max_samples(p0.geo, Sf, tile)
            fidx = torch.empty((B, H, Mf), dtype=torch.int32, device=dev)
            santa.santa_decode_attention_flash(p0.geo, p0.q, p0.K, p0.V, p0.seqlens, Sf, tile, args.seed, 0,
                                               p0.out, fidx, fws, stream)
            torch.cuda.synchronize()
            ii = fidx.cpu().numpy()
            fu = sum(len(np.unique(ii[b, g * G:(g + 1) * G])) for b in range(B) for g in range(Hkv))
            fkb, fvb, fqo = algorithmic_bytes([n] * B, Hkv, d, 2, float(fu), B, H)

            def flashp(i, Sf=Sf, tile=tile, fws=fws):
                p = probs[i % NR]
                santa.santa_decode_attention_flash(p.geo, p.q, p.K, p.V, p.seqlens, Sf, tile, args.seed, i, p.out,
                                                   None, fws, stream)
            for i in range(args.warmup):
                flashp(i)
            t = max_over_ranks(timed_loop(flashp, args.steps))
            flash[f"S{Sf}_tile{tile}"] = {"us_per_step": round(t * 1e3, 2),
                                          "GBps": round((fkb + fvb + fqo) / (t * 1e-3) / 1e9, 1),
                                          "frac": round((fkb + fvb + fqo) / (t * 1e-3) / 1e9 / peak, 4),
                                          "rows_per_head": Mf, "unique_rows": fu, "launches_per_step": 2}
            del fws
        res["flash"] = flash
        # (2) isolated single-step latency, the paper's protocol (flush write before each step)
        iso = []
        for i in range(args.steps):
            flush.zero_()
            a, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            step(i)
            b_.record(stream)
            torch.cuda.synchronize()
            iso.append(a.elapsed_time(b_))
        res["isolated_latency_us"] = {"mean": round(float(np.mean(iso)) * 1e3, 2),
                                      "median": round(float(np.median(iso)) * 1e3, 2),
                                      "p10": round(float(np.percentile(iso, 10)) * 1e3, 2),
                                      "p90": round(float(np.percentile(iso, 90)) * 1e3, 2),
                                      "protocol": "512 MiB L2-flush write, events around one call (P:1762-1777)"}
        # (3) in-repo dense exact decode, identical protocols
        dws = santa.workspace(p0.geo, 1, dev)

        def dense(i):
            p = probs[i % NR]
            santa.santa_dense_reference(p.geo, p.q, p.K, p.V, p.seqlens, p.out, dws, stream)
        for i in range(args.warmup):
            dense(i)
        dms = max_over_ranks(timed_loop(dense, args.steps))
        dbytes = 2 * kb + qo
        res["dense_reference"] = {"us": round(dms * 1e3, 2), "GBps": round(dbytes / (dms * 1e-3) / 1e9, 1),
                                  "santa_speedup": round(dms / ms, 3)}
        # (4) CUDA-graph replay of NR steps (launch overhead removed)
        try:
            g = torch.cuda.CUDAGraph()
            s2 = torch.cuda.Stream()
            s2.wait_stream(stream)
            with torch.cuda.stream(s2):
                for i in range(NR):
                    p = probs[i]
                    santa.santa_decode_attention(p.geo, p.q, p.K, p.V, p.seqlens, args.S, args.mode, args.seed, 0,
                                                 p.out, None, ws, s2)
            torch.cuda.synchronize()
            with torch.cuda.graph(g):
                cs = torch.cuda.current_stream()
                for i in range(NR):
                    p = probs[i]
                    santa.santa_decode_attention(p.geo, p.q, p.K, p.V, p.seqlens, args.S, args.mode, args.seed, 0,
                                                 p.out, None, ws, cs)
            reps = max(1, args.steps // NR)
            gms = timed_loop(lambda i: g.replay(), reps) / NR
            res["graph_replay_us"] = round(gms * 1e3, 2)
        except Exception as ex:  # graph capture is an extra, never the headline
            res["graph_replay_us"] = f"unavailable: {type(ex).__name__}: {ex}"[:200]
        # (5) end to end through the host-buffer C-ABI entry point: every step copies its packed
        # pinned [q | k_new | v_new] to the device (one H2D), appends the token to the cache, decodes,
        # and copies out back to pinned host memory (one D2H); K steps back-to-back, asynchronous,
        # CUDA events on the stream around all of them (+ the final sync inside the region)
        qkv_elems = B * H * d + 2 * B * Hkv * d
        qkvh = torch.randn(qkv_elems).to(torch.bfloat16).pin_memory()
        qkvh[:B * H * d].copy_(p0.q.reshape(-1).cpu())
        qkvd = torch.empty(qkv_elems, dtype=torch.bfloat16, device=dev)
        outh = torch.empty(B * H * d, dtype=torch.bfloat16).pin_memory()
        od = torch.empty_like(p0.q)

        def e2e_step(i):
            p = probs[i % NR]
            santa.santa_decode_step_host_packed(p.geo, qkvh, qkvd, p.K, p.V, p.seqlens, args.S, args.mode, args.seed,
                                                i, od, outh, ws, synchronize=False, stream=stream)
        for i in range(args.warmup):
            e2e_step(i)
        torch.cuda.synchronize()
        ems = max_over_ranks(timed_loop(e2e_step, args.steps))
        res["e2e"] = {"value": round(world * bytes_step / (ems * 1e-3) / 1e9, 2), "unit": "GB/s",
                      "us_per_step": round(ems * 1e3, 2),
                      "h2d_bytes_per_step": qkvh.numel() * 2, "d2h_bytes_per_step": outh.numel() * 2,
                      "path": "santa_decode_step_host_packed with pinned host buffers: per step the staging kernel "
                              "reads [q|k_new|v_new] from pinned host memory (zero copy) and appends the KV rows, "
                              "decode, the sampler writes out into pinned host memory; back-to-back asynchronous "
                              "steps, CUDA events (the staging kernel's PCIe reads are PDL-overlapped with the "
                              "previous step's sampler; a loop that syncs between steps measures "
                              "sync_call_latency_us)"}
        # the synchronous single-call latency of the same API (host wall clock incl. the stream sync)
        et = []
        for i in range(args.warmup + args.steps):
            p = probs[i % NR]
            t0 = time.perf_counter()
            santa.santa_decode_step_host_packed(p.geo, qkvh, qkvd, p.K, p.V, p.seqlens, args.S, args.mode, args.seed,
                                                i, od, outh, ws, synchronize=True, stream=stream)
            if i >= args.warmup:
                et.append(time.perf_counter() - t0)
        res["e2e"]["sync_call_latency_us"] = round(float(np.median(et)) * 1e6, 2)

    if not args.no_extras and args.batch == 1 and not args.page_size:
        if not args.no_config3:
            res["config3"] = config3(args, dev, stream, timed_loop, max_over_ranks, peak, world)
        if world == 1:
            res["config4_per_rank"] = config4(args, dev, stream, timed_loop, peak)
            res["config4_per_rank"]["peer_exchange_emulated"] = peer_exchange_emulated(args, dev, timed_loop)
            res["config5"] = config5(args, dev, stream, timed_loop, peak)
        else:
            res["config3_strong"] = config3_strong(args, dev, stream, timed_loop, max_over_ranks, peak, world, rank)
            res["config4_seqshard"] = config4_seqshard(args, dev, stream, timed_loop, max_over_ranks, peak, world,
                                                       rank)
    if world > 1:
        res["distributed"] = {"backend": args.dist_backend, "world": world,
                              "nccl_version": ".".join(map(str, torch.cuda.nccl.version()))
                              if args.dist_backend == "nccl" else None,
                              "nccl_debug": os.environ.get("NCCL_DEBUG")}
    if not args.no_extras and not args.no_baselines and rank == 0 and args.batch == 1 and not args.page_size:
        res["library_baselines"] = library_baselines(probs, NR, local_loop, args)
        d = res["library_baselines"]
        for k in ("flashinfer_decode_us", "flash_attn_2_decode_us", "torch_sdpa_us"):
            if isinstance(d.get(k), float):
                d[k.replace("_us", "_over_santa")] = round(d[k] / ms / 1e3, 3)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        res["cpu_baseline"] = cpu_baseline(probs[0].inp, args, bytes_step)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
