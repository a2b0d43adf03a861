"""One small call of every libsanta kernel family, for compute-sanitizer (tools/sanitize.sh and
tests/test_gpu_sanitize.py).  Shapes are tiny but span several chunks, a ragged tail, an odd
chunk-stat stride and every decode path; results are not checked here (the parity tests do that)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2605_01910_b200 as santa  # noqa: E402
from paper_2605_01910_b200 import sharding  # noqa: E402
import santa_inputs as si  # noqa: E402


def cuda(inp):
    for k in ("q", "K", "V", "seqlens", "K_pool", "V_pool", "page_table", "Kt"):
        v = getattr(inp, k)
        if v is not None:
            setattr(inp, k, v.cuda())
    return inp


def main():
    which = sys.argv[1].split(",") if len(sys.argv) > 1 else ["all"]
    run = lambda name: "all" in which or name in which  # noqa: E731
    inp = cuda(si.make_decode_inputs(2, 16, 4, 128, [1500, 700], dtype="bf16", seed=1, page_size=64))
    S = 64
    if run("decode"):
        for path in ("two_kernel", "step", "step_tc"):
            santa.decode(inp.q, inp.K, inp.V, inp.seqlens, S, "stratified", 3, return_idx=True, path=path)
        santa.decode(inp.q, inp.K_pool, inp.V_pool, inp.seqlens, S, "systematic", 3, page_table=inp.page_table,
                     page_size=64, max_seqlen=1536, return_idx=True)
        odd = cuda(si.make_decode_inputs(1, 8, 2, 128, [20000], dtype="bf16", seed=2))
        santa.decode(odd.q, odd.K, odd.V, odd.seqlens, 96, "iid", 3, return_idx=True)
        f32 = cuda(si.make_decode_inputs(1, 4, 4, 64, [1000], dtype="f32", seed=3))
        santa.decode(f32.q, f32.K, f32.V, f32.seqlens, 16, "systematic", 3, return_idx=True)
    if run("prop"):
        santa.decode_prop(inp.q, inp.K, inp.V, inp.seqlens, S, seed=3, return_idx=True)
    if run("flash"):
        santa.decode_flash(inp.q, inp.K, inp.V, inp.seqlens, 256, 256, seed=3, return_idx=True)
    if run("dense"):
        santa.dense(inp.q, inp.K, inp.V, inp.seqlens)
    if run("bernoulli"):
        b = cuda(si.make_decode_inputs(2, 16, 4, 128, [1024, 700], dtype="bf16", seed=4, workload="lognormal",
                                       feature_major=True))
        geo = santa.make_geometry(b.q, 4, b.Kt.shape[3])
        ws = santa.workspace(geo, S)
        sc = torch.zeros(2, 16, b.Kt.shape[3], device="cuda")
        santa.santa_bernoulli_scores(geo, b.q, b.Kt, b.seqlens, 8, 1, 1, 5, 0, sc, None, ws)
        out = torch.empty_like(b.q)
        santa.santa_decode_attention_bernoulli(geo, b.q, b.Kt, b.V, b.seqlens, 8, 1, 1, S, "stratified", 5, 0, out,
                                               None, ws)
    if run("seqshard"):
        be = sharding.CudaBackend()
        st = be.stats(inp.q, inp.K, inp.seqlens, 4, S)
        off = torch.zeros(2, dtype=torch.int32, device="cuda")
        be.sample_gather(torch.stack([st, st]), 0, 2, off, inp.V, inp.seqlens, S, "stratified", 3, 0,
                         return_idx=True)
    if run("host"):
        geo = santa.make_geometry(inp.q, 4, 1536)
        ws = santa.workspace(geo, S)
        qkv_h = torch.zeros(inp.q.numel() + 2 * 2 * 4 * 128, dtype=torch.bfloat16).pin_memory()
        qkv_d = torch.empty(qkv_h.numel(), dtype=torch.bfloat16, device="cuda")
        K, V = inp.K.clone(), inp.V.clone()
        K2 = torch.zeros(2, 4, 1536, 128, dtype=torch.bfloat16, device="cuda")
        V2 = torch.zeros_like(K2)
        K2[:, :, :1500] = K
        V2[:, :, :1500] = V
        out_h = torch.empty(inp.q.shape, dtype=torch.bfloat16).pin_memory()
        out_d = torch.empty_like(inp.q)
        santa.santa_decode_step_host_packed(geo, qkv_h, qkv_d, K2, V2, inp.seqlens, S, "stratified", 3, 0, out_d,
                                            out_h, ws)
    torch.cuda.synchronize()
    print("sanitize driver done:", ",".join(which))


if __name__ == "__main__":
    main()
