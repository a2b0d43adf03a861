"""Decode-loop integration (-m gpu): the KV append of the current token fused
into the decode step (santa_decode_attention_append) and per-layer sample budgets
(santa_decode_attention_layer, App. K).  The appended step must equal "append with
torch, then santa_decode_attention" bit for bit (same kernels read the same cache), write exactly
the new rows, and match the oracle (exemption rule, reading #19)."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

import santa_inputs as si  # noqa: E402

try:
    import paper_2605_01910_b200 as santa  # noqa: E402
    from gpu_helpers import check_parity, to_cuda  # noqa: E402
except ImportError:  # library not built: the gpu tests must fail loudly, not skip
    santa = None


@pytest.fixture(autouse=True)
def _need_lib():
    assert santa is not None, "libsanta.so not built"
    assert torch.cuda.is_available(), "no CUDA device"


def _new_rows(B, Hkv, d, dtype, seed):
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    k = torch.randn(B, Hkv, d, generator=g, device="cuda").to(dtype)
    v = torch.randn(B, Hkv, d, generator=g, device="cuda").to(dtype)
    return k, v


@pytest.mark.parametrize("B,H,n,S,want_path", [(2, 32, [3000, 1501], 128, "two_kernel"),
                                               (1, 32, [4096], 256, "two_kernel"),
                                               (32, 32, [2048] * 32, 64, "two_kernel")])
def test_append_equals_torch_append_then_decode(B, H, n, S, want_path):
    inp = to_cuda(si.make_decode_inputs(B, H, 8, 128, n, dtype="bf16", seed=71))
    geo = santa.make_geometry(inp.q, 8, inp.K.shape[2])
    assert santa.santa_auto_path(geo, S) == want_path
    k_new, v_new = _new_rows(B, 8, 128, inp.K.dtype, 72)
    # reference: write the rows with torch, then the plain decode step
    K_ref, V_ref = inp.K.clone(), inp.V.clone()
    for b, nb in enumerate(n):
        K_ref[b, :, nb - 1] = k_new[b]
        V_ref[b, :, nb - 1] = v_new[b]
    out_ref, idx_ref = santa.decode(inp.q, K_ref, V_ref, inp.seqlens, S, "stratified", 5, 2, return_idx=True)
    # the fused path on a cache whose new-token slots hold garbage
    K, V = inp.K.clone(), inp.V.clone()
    for b, nb in enumerate(n):
        K[b, :, nb - 1] = 1e4
        V[b, :, nb - 1] = -1e4
    out, idx = santa.decode_append(inp.q, K, V, k_new, v_new, inp.seqlens, S, "stratified", 5, 2, return_idx=True)
    torch.cuda.synchronize()
    assert torch.equal(K, K_ref) and torch.equal(V, V_ref)    # exactly the new rows were written
    assert torch.equal(idx, idx_ref) and torch.equal(out, out_ref)
    inp.K, inp.V = K, V
    sub = si.DecodeInputs(q=inp.q[:1], K=K[:1], V=V[:1], seqlens=inp.seqlens[:1], n_heads=H, n_kv_heads=8,
                          head_dim=128, dtype="bf16")
    check_parity(sub, out[:1], idx[:1], S, "stratified", 5, 2)


def test_append_paged_cache():
    """Pages of 64 keys (the fused producer path writes through the page table)."""
    n = [2000, 777]
    inp = to_cuda(si.make_decode_inputs(2, 16, 4, 128, n, dtype="bf16", seed=73, page_size=64))
    k_new, v_new = _new_rows(2, 4, 128, inp.K.dtype, 74)
    Kp, Vp = inp.K_pool.clone(), inp.V_pool.clone()
    geo = santa.make_geometry(inp.q, 4, inp.page_table.shape[1] * 64, inp.page_table, 64)
    ws = santa.workspace(geo, 96)
    out = torch.empty_like(inp.q)
    idx = torch.empty(2, 16, 96, dtype=torch.int32, device="cuda")
    santa.santa_decode_attention_append(geo, inp.q, Kp, Vp, k_new, v_new, inp.seqlens, 96, "systematic", 3, 0, out,
                                        idx, ws)
    torch.cuda.synchronize()
    tab = inp.page_table.cpu()
    for b, nb in enumerate(n):
        t = nb - 1
        page = int(tab[b, t // 64])
        assert torch.equal(Kp[page, :, t % 64], k_new[b]) and torch.equal(Vp[page, :, t % 64], v_new[b])
    K2, V2 = inp.K.clone(), inp.V.clone()
    for b, nb in enumerate(n):
        K2[b, :, nb - 1] = k_new[b]
        V2[b, :, nb - 1] = v_new[b]
    sub = si.DecodeInputs(q=inp.q, K=K2, V=V2, seqlens=inp.seqlens, n_heads=16, n_kv_heads=4, head_dim=128,
                          dtype="bf16")
    check_parity(sub, out, idx, 96, "systematic", 3, 0)


def test_per_layer_schedule():
    """santa_decode_attention_layer(layer l) == santa_decode_attention with S = S_l and Philox offset
    offset * n_layers + l, bit for bit; one workspace of santa_schedule_workspace_bytes serves every
    layer; an out-of-range layer launches nothing."""
    Ss = [8, 64, 256, 16]
    sched = santa.make_schedule(Ss)
    inp = to_cuda(si.make_decode_inputs(2, 32, 8, 128, [5000, 3333], dtype="bf16", seed=75))
    geo = santa.make_geometry(inp.q, 8, inp.K.shape[2])
    ws = torch.zeros(santa.santa_schedule_workspace_bytes(geo, sched), dtype=torch.uint8, device="cuda")
    step = 11
    for layer, S in enumerate(Ss):
        out = torch.empty_like(inp.q)
        idx = torch.empty(2, 32, S, dtype=torch.int32, device="cuda")
        santa.santa_decode_attention_layer(geo, sched, layer, inp.q, inp.K, inp.V, None, None, inp.seqlens,
                                           "stratified", 9, step, out, idx, ws)
        ref_out, ref_idx = santa.decode(inp.q, inp.K, inp.V, inp.seqlens, S, "stratified", 9,
                                        step * len(Ss) + layer, return_idx=True)
        torch.cuda.synchronize()
        assert torch.equal(idx, ref_idx) and torch.equal(out, ref_out), layer
    with pytest.raises(santa.SantaError):
        santa.santa_decode_attention_layer(geo, sched, 4, inp.q, inp.K, inp.V, None, None, inp.seqlens,
                                           "stratified", 9, step, out, idx, ws)


def test_prepared_decode_equals_the_plain_call():
    """prepare_decode (arguments marshalled once, launch(offset) per step) launches exactly the
    santa_decode_attention_path call: same bits for every offset."""
    inp = to_cuda(si.make_decode_inputs(2, 32, 8, 128, [4000, 2500], dtype="bf16", seed=76))
    geo = santa.make_geometry(inp.q, 8, inp.K.shape[2])
    ws = santa.workspace(geo, 128)
    out = torch.empty_like(inp.q)
    idx = torch.empty(2, 32, 128, dtype=torch.int32, device="cuda")
    launch = santa.prepare_decode(geo, inp.q, inp.K, inp.V, inp.seqlens, 128, "systematic", 4, out, idx, ws)
    for off in (0, 5, 123456789):
        launch(off)
        ref_out, ref_idx = santa.decode(inp.q, inp.K, inp.V, inp.seqlens, 128, "systematic", 4, off, return_idx=True)
        torch.cuda.synchronize()
        assert torch.equal(idx, ref_idx) and torch.equal(out, ref_out), off


@pytest.mark.parametrize("dtype,d,H,Hkv", [("f16", 64, 16, 2), ("bf16", 128, 8, 8)])
def test_append_dtype_shape_variants(dtype, d, H, Hkv):
    """The fused append on fp16 / d = 64 / G = 8 and on G = 1 geometries."""
    n = [1700, 900]
    inp = to_cuda(si.make_decode_inputs(2, H, Hkv, d, n, dtype=dtype, seed=77))
    k_new, v_new = _new_rows(2, Hkv, d, inp.K.dtype, 78)
    K_ref, V_ref = inp.K.clone(), inp.V.clone()
    for b, nb in enumerate(n):
        K_ref[b, :, nb - 1] = k_new[b]
        V_ref[b, :, nb - 1] = v_new[b]
    out_ref, idx_ref = santa.decode(inp.q, K_ref, V_ref, inp.seqlens, 64, "stratified", 8, 0, return_idx=True)
    K, V = inp.K.clone(), inp.V.clone()
    out, idx = santa.decode_append(inp.q, K, V, k_new, v_new, inp.seqlens, 64, "stratified", 8, 0, return_idx=True)
    torch.cuda.synchronize()
    assert torch.equal(K, K_ref) and torch.equal(V, V_ref)
    assert torch.equal(idx, idx_ref) and torch.equal(out, out_ref)


def test_pdl_chained_steps_see_the_preceding_kernels_writes():
    """PDL (the score pass, the dense kernel and the Bernoulli weights kernel are launched with
    programmatic stream serialization and wait in one thread after their barrier set-up): a torch
    kernel that writes q, K and V immediately before each call, with no sync, must be seen by that
    call -- 12 back-to-back steps on changing inputs equal the same steps run one at a time with a
    device sync before each."""
    B, H, Hkv, d, n, S = 1, 32, 8, 128, [8192], 256
    base = to_cuda(si.make_decode_inputs(B, H, Hkv, d, n, dtype="bf16", seed=81))
    geo = santa.make_geometry(base.q, Hkv, n[0])
    ws = santa.workspace(geo, S)
    q, K, V = base.q.clone(), base.K.clone(), base.V.clone()
    g = torch.Generator(device="cuda").manual_seed(82)
    qs = [torch.randn(q.shape, generator=g, device="cuda").to(q.dtype) for _ in range(12)]
    ks = [torch.randn(K.shape[:-2] + (64, d), generator=g, device="cuda").to(K.dtype) for _ in range(12)]

    def run(i, out, sync):
        if sync:
            torch.cuda.synchronize()
        q.copy_(qs[i])                      # producer kernels right before the call
        K[:, :, :64].copy_(ks[i])
        V[:, :, 64:128].copy_(ks[i])
        santa.santa_decode_attention(geo, q, K, V, base.seqlens, S, "stratified", 9, i, out, None, ws)
        d_out = out.clone()
        santa.santa_dense_reference(geo, q, K, V, base.seqlens, out, ws)
        return d_out, out.clone()

    outs = [torch.empty_like(q) for _ in range(12)]
    fast = [run(i, outs[i], False) for i in range(12)]
    ref = [run(i, outs[i], True) for i in range(12)]
    torch.cuda.synchronize()
    for i in range(12):
        assert torch.equal(fast[i][0], ref[i][0]), i
        assert torch.equal(fast[i][1], ref[i][1]), i
