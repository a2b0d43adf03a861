"""Times the paper's comparison systems (FlashInfer decode, FlashAttention-2 decode) and torch
SDPA on the config-2 decode step, with the same protocol as bench.py (back-to-back over rotating
KV caches > L2), for context next to the in-repo kernels.  Library kernels, not part of the
product; failures are reported, not fatal."""
import json
import sys
import time

import torch

B, H, Hkv, d, n = 1, 32, 8, 128, 32768
NR, K, W = 4, 50, 10


def timed(fn):
    for i in range(W):
        fn(i)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(K):
        fn(i)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / K * 1e3


def main():
    dev = "cuda"
    g = torch.Generator(device=dev).manual_seed(0)
    qs = [torch.randn(B, H, d, generator=g, device=dev).bfloat16() for _ in range(NR)]
    # sequence-major caches as the libraries expect: [B, n, Hkv, d]
    Ks = [torch.randn(B, n, Hkv, d, generator=g, device=dev).bfloat16() for _ in range(NR)]
    Vs = [torch.randn(B, n, Hkv, d, generator=g, device=dev).bfloat16() for _ in range(NR)]
    res = {}
    kv_bytes = 2 * B * n * Hkv * d * 2
    try:
        from flash_attn import flash_attn_with_kvcache
        sl = torch.full((B,), n, dtype=torch.int32, device=dev)
        us = timed(lambda i: flash_attn_with_kvcache(qs[i % NR].unsqueeze(1), Ks[i % NR], Vs[i % NR],
                                                     cache_seqlens=sl))
        res["flash_attn_2_decode_us"] = round(us, 2)
    except Exception as e:  # noqa: BLE001
        res["flash_attn_2_decode_us"] = f"unavailable: {type(e).__name__}: {str(e)[:160]}"
    try:
        import flashinfer
        t0 = time.time()
        us = timed(lambda i: flashinfer.single_decode_with_kv_cache(qs[i % NR][0], Ks[i % NR][0], Vs[i % NR][0]))
        res["flashinfer_decode_us"] = round(us, 2)
        res["flashinfer_first_call_s"] = round(time.time() - t0, 1)
    except Exception as e:  # noqa: BLE001
        res["flashinfer_decode_us"] = f"unavailable: {type(e).__name__}: {str(e)[:160]}"
    try:
        Kt = [k.transpose(1, 2).contiguous() for k in Ks]
        Vt = [v.transpose(1, 2).contiguous() for v in Vs]
        us = timed(lambda i: torch.nn.functional.scaled_dot_product_attention(
            qs[i % NR].unsqueeze(2), Kt[i % NR], Vt[i % NR], enable_gqa=True))
        res["torch_sdpa_us"] = round(us, 2)
    except Exception as e:  # noqa: BLE001
        res["torch_sdpa_us"] = f"unavailable: {type(e).__name__}: {str(e)[:160]}"
    res["kv_bytes"] = kv_bytes
    for k in list(res):
        if k.endswith("_us") and isinstance(res[k], float):
            res[k.replace("_us", "_GBps")] = round(kv_bytes / (res[k] * 1e-6) / 1e9, 1)
    print(json.dumps(res))


if __name__ == "__main__":
    sys.exit(main())
