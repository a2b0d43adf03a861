"""GPU vs oracle parity through the C-ABI (-m gpu).  Sizes span several 256-key chunks and a
ragged tail; the full BASELINE config-2 size is checked on sampled heads."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

import santa_inputs as si  # noqa: E402
from oracle import santa_oracle as o  # noqa: E402

try:
    import paper_2605_01910_b200 as santa  # noqa: E402
    from gpu_helpers import TOL, check_parity, gpu_decode, oracle_decode, to_cuda  # noqa: E402
except ImportError:  # library not built: the gpu tests must fail loudly, not skip
    santa = None


@pytest.fixture(autouse=True)
def _need_lib():
    assert santa is not None, "libsanta.so not built"
    assert torch.cuda.is_available(), "no CUDA device"


REPORT = []


def test_philox_device_matches_kat_and_oracle():
    raw = torch.zeros(4, dtype=torch.int32, device="cuda")
    u = torch.empty(1000, dtype=torch.float64, device="cuda")
    for ctr_key, want in [((0, 0, 0, 0, 0, 0), (0x6627e8d5, 0xe169c58d, 0xbc57ac4c, 0x9b00dbd8)),
                          ((0xffffffff,) * 6, (0x408f276d, 0x41c83b0e, 0xa20bc7c6, 0x6d5451fd)),
                          ((0x243f6a88, 0x85a308d3, 0x13198a2e, 0x03707344, 0xa4093822, 0x299f31d0),
                           (0xd16cfe09, 0x94fdcceb, 0x5001e420, 0x24126ea1))]:
        santa.santa_philox_uniforms(0, 0, 1, 0, 0, 4, u, ctr_key, raw)
        torch.cuda.synchronize()
        got = tuple(int(x) & 0xffffffff for x in raw.cpu().tolist())
        assert got == want
    for seed, off, tag, h, b in [(0x5A17A, 0, 1, 3, 7), (2 ** 40 + 5, 123, 3, 17, 0), (1, 2 ** 33 + 9, 2, 0, 31)]:
        santa.santa_philox_uniforms(seed, off, tag, h, b, 1000, u)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(u.cpu().numpy(), o.philox_uniforms(seed, off, tag, h, b, np.arange(1000)))


@pytest.mark.parametrize("mode", o.MODES)
def test_c1_fp32_single_head(mode):
    """BASELINE config 1: single head, n_k=1024, d=64, fp32, S=16 (systematic; all modes)."""
    inp = to_cuda(si.make_decode_inputs(1, 1, 1, 64, 1024, dtype="f32", seed=1))
    out, idx = gpu_decode(inp, 16, mode, seed=0x5A17A)
    REPORT.append(("c1", mode, check_parity(inp, out, idx, 16, mode, 0x5A17A)))


@pytest.mark.parametrize("path", ["step", "step_tc", "two_kernel"])
@pytest.mark.parametrize("mode", o.MODES)
@pytest.mark.parametrize("paged", [False, True])
def test_bf16_gqa_ragged(mode, paged, path):
    """Llama GQA shape (H=32, H_kv=8, d=128, bf16), ragged seqlens spanning many chunks and
    partial tails; contiguous and shuffled paged (P=64) layouts; both execution paths."""
    inp = si.make_decode_inputs(2, 32, 8, 128, [4097, 1000], dtype="bf16", seed=2,
                                page_size=(128 if path == "step_tc" else 64) if paged else 0)
    inp = to_cuda(inp)
    out, idx = gpu_decode(inp, 256, mode, seed=11, offset=3, paged=paged, path=path)
    REPORT.append(("gqa", mode, paged, path, check_parity(inp, out, idx, 256, mode, 11, 3)))


@pytest.mark.parametrize("path", ["auto", "step", "step_tc"])
@pytest.mark.parametrize("dtype,d,H,Hkv", [("f16", 64, 16, 2), ("bf16", 64, 8, 8), ("bf16", 128, 8, 4),
                                            ("f32", 128, 16, 8), ("bf16", 128, 4, 2), ("f16", 128, 32, 4)])
def test_dtype_shape_variants(dtype, d, H, Hkv, path):
    """dtypes, head dims and GQA group sizes G = 8, 1, 2, 2, 8 on every decode path (the step
    kernels take bf16/fp16 only: fp32 must be refused, not silently rerouted)."""
    inp = to_cuda(si.make_decode_inputs(2, H, Hkv, d, [777, 2048], dtype=dtype, seed=3, workload="temp4"))
    if dtype == "f32" and path != "auto":
        with pytest.raises(santa.SantaError) as e:
            gpu_decode(inp, 64, "systematic", seed=5, path=path)
        assert e.value.status == 5  # SANTA_ERR_UNSUPPORTED
        return
    out, idx = gpu_decode(inp, 64, "systematic", seed=5, path=path)
    check_parity(inp, out, idx, 64, "systematic", 5)


@pytest.mark.parametrize("workload", ["temp4", "sink"])
def test_peaked_workloads(workload):
    inp = to_cuda(si.make_decode_inputs(1, 32, 8, 128, 3000, dtype="bf16", seed=4, workload=workload))
    for mode in o.MODES:
        out, idx = gpu_decode(inp, 128, mode, seed=9)
        check_parity(inp, out, idx, 128, mode, 9)


@pytest.mark.parametrize("path", ["step", "step_tc", "two_kernel"])
def test_edge_cases_small_and_large_budgets(path):
    # seqlen 1, S = 1, S > n (with replacement), non-power-of-two S, big max_seqlen padding
    inp = to_cuda(si.make_decode_inputs(3, 8, 2, 128, [1, 17, 300], dtype="bf16", seed=5))
    for S in (1, 3, 100, 1024):
        for mode in o.MODES:
            out, idx = gpu_decode(inp, S, mode, seed=S, path=path)
            check_parity(inp, out, idx, S, mode, S)
            assert torch.all(idx[0] == 0)
    out1, idx1 = gpu_decode(inp, 64, "stratified", seed=1, path=path)
    # the same sequences inside a cache padded to max_seqlen = 5000 (20 chunks, mostly empty)
    pad = torch.nn.functional.pad
    big = si.DecodeInputs(q=inp.q, K=pad(inp.K, (0, 0, 0, 4700)).contiguous(),
                          V=pad(inp.V, (0, 0, 0, 4700)).contiguous(), seqlens=inp.seqlens, n_heads=8,
                          n_kv_heads=2, head_dim=128, dtype="bf16")
    out2, idx2 = gpu_decode(big, 64, "stratified", seed=1, path=path)
    assert torch.equal(idx1, idx2) and torch.equal(out1, out2)


@pytest.mark.parametrize("path", ["step", "step_tc", "two_kernel"])
def test_empty_sequence_sets_flag_and_zeroes(path):
    inp = to_cuda(si.make_decode_inputs(2, 8, 2, 128, [5, 40], dtype="bf16", seed=6))
    inp.seqlens[0] = 0
    geo = santa.make_geometry(inp.q, 2, 40)
    ws = santa.workspace(geo, 8)
    out = torch.full_like(inp.q, 7.0)
    idx = torch.empty((2, 8, 8), dtype=torch.int32, device="cuda")
    santa.santa_decode_attention_path(geo, inp.q, inp.K, inp.V, inp.seqlens, 8, "stratified", 1, 0, out, idx, ws,
                                      path)
    flags = santa.santa_read_error_flags(ws)
    assert flags & santa.FLAG_EMPTY_SEQ
    assert torch.all(out[0] == 0) and torch.all(idx[0] == -1)
    assert torch.all(idx[1] >= 0) and torch.all(idx[1] < 40)
    inp.seqlens[0] = 5
    santa.santa_decode_attention_path(geo, inp.q, inp.K, inp.V, inp.seqlens, 8, "stratified", 1, 0, out, idx, ws,
                                      path)
    assert santa.santa_read_error_flags(ws) == 0


def test_invalid_arguments_launch_nothing():
    inp = to_cuda(si.make_decode_inputs(1, 8, 2, 128, 64, dtype="bf16", seed=7))
    geo = santa.make_geometry(inp.q, 2, 64)
    ws = santa.workspace(geo, 8)
    out = torch.full_like(inp.q, 3.0)
    for kwargs, status in [(dict(S=0), 3), (dict(mode=7), 1), (dict(ws=ws[:100]), 6), (dict(ws=ws[1:]), 6)]:
        args = dict(S=8, mode=1, ws=ws)
        args.update(kwargs)
        with pytest.raises(santa.SantaError) as e:
            santa.santa_decode_attention(geo, inp.q, inp.K, inp.V, inp.seqlens, args["S"], args["mode"], 1, 0, out,
                                         None, args["ws"])
        assert e.value.status == status
    torch.cuda.synchronize()
    assert torch.all(out == 3.0)


@pytest.mark.parametrize("path", ["step", "step_tc"])
def test_forced_step_paths_refuse_long_contexts(path):
    """the step kernels' sampler keeps <= 1024 chunk statistics per head in
    registers, so a forced step path on max_seqlen > 65,536 must return SANTA_ERR_UNSUPPORTED and
    launch nothing (AUTO takes the two-kernel path there)."""
    n = 65536 + 64
    inp = to_cuda(si.make_decode_inputs(1, 8, 2, 128, n, dtype="bf16", seed=7))
    geo = santa.make_geometry(inp.q, 2, n)
    ws = santa.workspace(geo, 64)
    out = torch.full_like(inp.q, 3.0)
    with pytest.raises(santa.SantaError) as e:
        santa.santa_decode_attention_path(geo, inp.q, inp.K, inp.V, inp.seqlens, 64, 1, 1, 0, out, None, ws, path)
    assert e.value.status == 5
    torch.cuda.synchronize()
    assert torch.all(out == 3.0)
    assert santa.santa_auto_path(geo, 64) == "two_kernel"
    got, idx = gpu_decode(inp, 64, "stratified", seed=1)   # AUTO on the same geometry works
    check_parity(inp, got, idx, 64, "stratified", seed=1)


def test_host_step_apis_validate_before_touching_the_cache():
    """santa_decode_step_host(_packed) run every decode check BEFORE the first copy or
    launch, so an invalid call (S too large, bad mode) leaves the K/V cache and outputs untouched."""
    B, H, Hkv, d = 1, 8, 2, 128
    inp = to_cuda(si.make_decode_inputs(B, H, Hkv, d, 300, dtype="bf16", seed=7))
    geo = santa.make_geometry(inp.q, Hkv, 300)
    ws = santa.workspace(geo, 8)
    K0, V0 = inp.K.clone(), inp.V.clone()
    qkv = torch.randn(B * H * d + 2 * B * Hkv * d).to(torch.bfloat16).pin_memory()
    out_h = torch.full((B * H * d,), 3.0, dtype=torch.bfloat16).pin_memory()
    dev = torch.empty(B * H * d + 2 * B * Hkv * d, dtype=torch.bfloat16, device="cuda")
    od = torch.full_like(inp.q, 3.0)
    for S, mode, status in [(5000, 1, 5), (8, 7, 1), (0, 1, 3)]:
        with pytest.raises(santa.SantaError) as e:
            santa.santa_decode_step_host_packed(geo, qkv, dev, inp.K, inp.V, inp.seqlens, S, mode, 1, 0, od, out_h, ws)
        assert e.value.status == status
        qh, kh, vh = (torch.randn(B, h_, d).to(torch.bfloat16).pin_memory() for h_ in (H, Hkv, Hkv))
        with pytest.raises(santa.SantaError) as e:
            santa.santa_decode_step_host(geo, qh, kh, vh, torch.empty_like(inp.q), torch.empty(B, Hkv, d, dtype=torch.bfloat16, device="cuda"),
                                         torch.empty(B, Hkv, d, dtype=torch.bfloat16, device="cuda"), inp.K, inp.V,
                                         inp.seqlens, S, mode, 1, 0, od, out_h, ws)
        assert e.value.status == status
    torch.cuda.synchronize()
    assert torch.equal(inp.K, K0) and torch.equal(inp.V, V0)
    assert torch.all(od == 3.0) and torch.all(out_h == 3.0)


def test_determinism_bitwise():
    inp = to_cuda(si.make_decode_inputs(2, 32, 8, 128, [3000, 2500], dtype="bf16", seed=8))
    a = gpu_decode(inp, 256, "stratified", seed=3)
    b = gpu_decode(inp, 256, "stratified", seed=3)
    assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1])
    c = gpu_decode(inp, 256, "stratified", seed=4)
    assert not torch.equal(a[1], c[1])


def test_paged_equals_contiguous():
    inp = si.make_decode_inputs(2, 16, 4, 128, [2000, 1234], dtype="bf16", seed=9, page_size=32)
    inp = to_cuda(inp)
    a = gpu_decode(inp, 128, "systematic", seed=1)
    b = gpu_decode(inp, 128, "systematic", seed=1, paged=True)
    assert torch.equal(a[1], b[1]) and torch.equal(a[0], b[0])


def test_systematic_count_invariant_on_gpu():
    """Every systematic count is floor or ceil of S p_j (p from the oracle's fp64 softmax),
    up to boundary-exempt samples."""
    inp = to_cuda(si.make_decode_inputs(1, 8, 2, 128, 500, dtype="bf16", seed=10, workload="temp4"))
    S = 64
    out, idx = gpu_decode(inp, S, "systematic", seed=2)
    q, K = o.to_f64(si.as_bits(inp.q)), o.to_f64(si.as_bits(inp.K))
    for h in range(8):
        p = o.softmax(o.scores(q[0, h], K[0, h // 4, :500], 1 / np.sqrt(128)))
        c = np.bincount(idx[0, h].cpu().numpy(), minlength=500)
        assert c.sum() == S
        assert np.sum((c < np.floor(S * p - 1e-6)) | (c > np.ceil(S * p + 1e-6))) <= 2


def test_full_size_config2_sampled_heads():
    """BASELINE config 2 at full size (32k, batch 1, S=256 stratified), in the launch
    configuration bench.py times (the single-launch step kernel); the oracle recomputes two
    kv-head groups (8 heads).  The two-kernel path must give the same indices."""
    inp = to_cuda(si.make_decode_inputs(1, 32, 8, 128, 32768, dtype="bf16", seed=0))
    out, idx = gpu_decode(inp, 256, "stratified", seed=0x5A17A, path="step")
    out2, idx2 = gpu_decode(inp, 256, "stratified", seed=0x5A17A, path="two_kernel")
    out3, idx3 = gpu_decode(inp, 256, "stratified", seed=0x5A17A, path="step_tc")
    # the tensor-core score stage sums the same bf16 products in another order (fp32): same indices
    # up to threshold-at-boundary cases
    assert (idx != idx3).float().mean().item() < 1e-3
    # the paths differ only in the in-chunk prefix encoding (fp32 vs 24-bit fixed point, reading #23):
    # indices may differ only where a threshold lies within ~2^-24 of a key boundary
    assert (idx != idx2).float().mean().item() < 1e-3
    for kvh in (0, 5):
        sub = si.DecodeInputs(q=inp.q[:, 4 * kvh:4 * kvh + 4].contiguous(), K=inp.K[:, kvh:kvh + 1].contiguous(),
                              V=inp.V[:, kvh:kvh + 1].contiguous(), seqlens=inp.seqlens, n_heads=4, n_kv_heads=1,
                              head_dim=128, dtype="bf16")
        for path, o_, i_ in (("step", out, idx), ("two_kernel", out2, idx2), ("step_tc", out3, idx3)):
            REPORT.append(("c2-full", kvh, path,
                           check_parity(sub, o_[:, 4 * kvh:4 * kvh + 4], i_[:, 4 * kvh:4 * kvh + 4], 256, "stratified",
                                        0x5A17A, head_offset=4 * kvh)))


def _step_tickets(ws, B, H, Hkv):
    """The step kernel's ticket words (santa_abi.cu layout(): flags | tickets | epoch, exit, heads)."""
    a256 = lambda x: (x + 255) // 256 * 256  # noqa: E731
    off = 256 + a256(B * Hkv * 4)
    words = ws[off:off + (2 + B * H) * 4].view(torch.int32)
    return int(words[0].item()), words[1:]


@pytest.mark.parametrize("B,n,S", [(1, 32768, 256), (4, [5000, 1, 2222, 4096], 1024), (3, [300, 700, 64], 16)])
def test_step_kernel_tickets_and_epoch(B, n, S):
    """Consecutive single-launch steps on one workspace: every ticket is back to zero after each
    launch, the epoch advances by one per launch, and every launch reproduces a fresh-workspace
    run (stale tagged words of earlier launches are never taken for current ones)."""
    inp = to_cuda(si.make_decode_inputs(B, 32, 8, 128, n, dtype="bf16", seed=21))
    geo = santa.make_geometry(inp.q, 8, int(inp.K.shape[2]))
    ws = santa.workspace(geo, S)
    out = torch.empty_like(inp.q)
    idx = torch.empty((B, 32, S), dtype=torch.int32, device="cuda")
    for rep, seed in enumerate([1, 2, 1, 3, 1]):
        santa.santa_decode_attention_path(geo, inp.q, inp.K, inp.V, inp.seqlens, S, "stratified", seed, 0, out, idx,
                                          ws, "step")
        torch.cuda.synchronize()
        epoch, tickets = _step_tickets(ws, B, 32, 8)
        assert epoch == rep + 1 and int(tickets.count_nonzero()) == 0, (rep, epoch)
        assert santa.santa_read_error_flags(ws) == 0
        ref_out, ref_idx = gpu_decode(inp, S, "stratified", seed, path="step")
        assert torch.equal(idx, ref_idx) and torch.equal(out, ref_out), rep


def test_batch_offset_and_head_offset_key_the_stream():
    """Philox is keyed by GLOBAL (b, h): a shard with offsets reproduces the full run's rows."""
    inp = to_cuda(si.make_decode_inputs(4, 16, 4, 128, 700, dtype="bf16", seed=11))
    full_out, full_idx = gpu_decode(inp, 64, "stratified", seed=5)
    sub = si.DecodeInputs(q=inp.q[2:4, 8:12].contiguous(), K=inp.K[2:4, 2:3].contiguous(),
                          V=inp.V[2:4, 2:3].contiguous(), seqlens=inp.seqlens[2:4].contiguous(), n_heads=4,
                          n_kv_heads=1, head_dim=128, dtype="bf16")
    o2, i2 = gpu_decode(sub, 64, "stratified", seed=5, head_offset=8, batch_offset=2)
    assert torch.equal(i2, full_idx[2:4, 8:12]) and torch.equal(o2, full_out[2:4, 8:12])


def test_dense_reference_parity():
    for dtype, d, H, Hkv, n in [("bf16", 128, 32, 8, [4097, 1000]), ("f32", 64, 1, 1, [1024, 3]),
                                ("f16", 64, 16, 2, [300, 2048])]:
        inp = to_cuda(si.make_decode_inputs(2, H, Hkv, d, n, dtype=dtype, seed=12, workload="temp4"))
        out = santa.dense(inp.q, inp.K, inp.V, inp.seqlens)
        torch.cuda.synchronize()
        ref = o.dense_decode(si.as_bits(inp.q), si.as_bits(inp.K), si.as_bits(inp.V), inp.seqlens.cpu().numpy())
        err = np.abs(out.float().cpu().numpy() - ref).max()
        # fp32 partials; bf16 output rounding |x| <= ~4 -> 2^-8 * 4
        assert err <= (2e-5 if dtype == "f32" else 2e-2), (dtype, err)


@pytest.mark.parametrize("mode", o.MODES)
def test_unbiasedness_gpu_3sigma(mode):
    """Mean of the GPU estimator over 1e4 seeds converges to dense AV within 3 sigma
    (Props); sigma from the exact per-scheme variance (reading #17)."""
    inp = to_cuda(si.make_decode_inputs(1, 4, 1, 128, 48, dtype="f32", seed=13, workload="temp4"))
    S, N = 8, 10000
    geo = santa.make_geometry(inp.q, 1, 48)
    ws = santa.workspace(geo, S)
    out = torch.empty_like(inp.q)
    acc = torch.zeros(4, 128, dtype=torch.float64, device="cuda")
    for seed in range(N):
        santa.santa_decode_attention(geo, inp.q, inp.K, inp.V, inp.seqlens, S, mode, seed, 0, out, None, ws)
        acc += out[0].double()
    mean = (acc / N).cpu().numpy()
    q, K, V = (o.to_f64(si.as_bits(t)) for t in (inp.q, inp.K, inp.V))
    zmax = 0.0
    for h in range(4):
        p = o.softmax(o.scores(q[0, h], K[0, 0, :48], 1 / np.sqrt(128)))
        if mode == "iid":
            var = o.var_iid_per_coord(p, V[0, 0, :48], S)
        elif mode == "stratified":
            var = o.var_stratified(p, V[0, 0, :48], S)[0]
        else:
            var = o.systematic_law(p, V[0, 0, :48], S)[1]
        z = (mean[h] - p @ V[0, 0, :48]) / np.sqrt(np.maximum(var, 1e-30) / N)
        z[var < 1e-20] = 0.0
        zmax = max(zmax, np.abs(z).max())
    assert zmax < 4.97   # Sidak-adjusted 3-sigma level over 4 x 128 coordinates (reading #17)


def test_report_mismatch_rates(capsys):
    with capsys.disabled():
        for r in REPORT:
            print("index parity", r)


def test_odd_chunk_strides_and_unaligned_stats_rows():
    """Chunk-stat rows of odd length (Cmax odd: a head's stats start 8-B but not 16-B aligned) with
    256 < chunks <= 512 per sequence (the sampler's paired 16-B stats loads): parity with the oracle."""
    inp = to_cuda(si.make_decode_inputs(3, 16, 4, 128, [20000, 16447, 19000], dtype="bf16", seed=63))
    out, idx = gpu_decode(inp, 192, "stratified", seed=5)
    REPORT.append(("odd-Cmax", 0, "auto", check_parity(inp, out, idx, 192, "stratified", 5)))


@pytest.mark.parametrize("B,n,units", [(1, 32768, [(0, 0), (0, 7)]), (4, [40000, 39001, 40000, 12345],
                                                                       [(0, 3), (1, 7), (3, 0)])])
def test_dense_reference_split_shapes(B, n, units):
    """The split-KV dense kernel in both of its shapes: config 2 (3 warps x 4 slots, 16-part LSE
    combine: ~19 CTAs per unit) and above 4 MiB of K+V per SM (5 warps x 2 slots, one combine CTA per
    head), against the fp64 dense oracle on sampled (b, kv-head) units incl. a ragged last stage."""
    inp = si.make_decode_inputs(B, 32, 8, 128, n, dtype="bf16", seed=14, workload="temp4", device="cuda")
    out = santa.dense(inp.q, inp.K, inp.V, inp.seqlens)
    torch.cuda.synchronize()
    lens = inp.seqlens.cpu().numpy()
    for b, kvh in units:
        hs = slice(4 * kvh, 4 * kvh + 4)
        ref = o.dense_decode(si.as_bits(inp.q[b:b + 1, hs]), si.as_bits(inp.K[b:b + 1, kvh:kvh + 1]),
                             si.as_bits(inp.V[b:b + 1, kvh:kvh + 1]), lens[b:b + 1])
        err = np.abs(out[b:b + 1, hs].float().cpu().numpy() - ref).max()
        assert err <= 2e-2, (b, kvh, err)


@pytest.mark.parametrize("paged", [False, True])
def test_large_batch_sampler_paged_and_ragged(paged):
    """The 4-CTA-per-SM sampler build (more than two sampler CTAs per SM: 12 x 32 = 384 heads) on a
    ragged batch, contiguous and through a 64-key page table: the same indices and outputs as the
    single-launch step kernel (independent sampler code), and oracle parity on sampled units incl. the
    shortest sequence."""
    n = [4096, 1500, 33, 4095, 64, 2047, 3000, 129, 4000, 1, 2500, 4096]
    inp = to_cuda(si.make_decode_inputs(12, 32, 8, 128, n, dtype="bf16", seed=91, workload="temp4",
                                        page_size=64 if paged else 0))
    S = 128
    out, idx = gpu_decode(inp, S, "stratified", seed=5, offset=2, paged=paged, path="two_kernel")
    out2, idx2 = gpu_decode(inp, S, "stratified", seed=5, offset=2, paged=paged, path="step")
    assert (idx != idx2).float().mean().item() < 2e-3
    G = 4
    for b, kvh in [(2, 0), (9, 3), (11, 7)]:
        sub = si.DecodeInputs(q=inp.q[b:b + 1, G * kvh:G * (kvh + 1)].contiguous(),
                              K=inp.K[b:b + 1, kvh:kvh + 1].contiguous(), V=inp.V[b:b + 1, kvh:kvh + 1].contiguous(),
                              seqlens=inp.seqlens[b:b + 1].contiguous(), n_heads=G, n_kv_heads=1, head_dim=128,
                              dtype="bf16")
        check_parity(sub, out[b:b + 1, G * kvh:G * (kvh + 1)], idx[b:b + 1, G * kvh:G * (kvh + 1)], S, "stratified",
                     5, 2, head_offset=G * kvh, batch_offset=b)


def test_seqshard_large_batch_sampler():
    """Sequence sharding with more sampler CTAs than two per SM (12 x 32 heads: the 4-per-SM build in
    phase 2, strata of other shards skipped): two simulated shards' merged indices equal the unsharded
    run and every stratum is owned by exactly one shard."""
    from paper_2605_01910_b200 import sharding
    n = [6000, 3001, 4096, 129, 5000, 6000, 2048, 777, 6000, 4500, 1000, 6000]
    B, H, Hkv, d, S = 12, 32, 8, 128, 256
    inp = to_cuda(si.make_decode_inputs(B, H, Hkv, d, n, dtype="bf16", seed=93))
    full_out, full_idx = gpu_decode(inp, S, "stratified", seed=8, offset=1)
    R = 2
    parts, owner = [], torch.zeros(B, H, S, dtype=torch.int32, device="cuda")
    merged = torch.full((B, H, S), -1, dtype=torch.int32, device="cuda")
    stats, shards = [], []
    for r in range(R):
        lo, ln = sharding.shard_ranges(inp.seqlens, r, R, "cuda")
        nloc = int(ln.max())
        Ks = torch.zeros(B, Hkv, nloc, d, dtype=inp.K.dtype, device="cuda")
        Vs = torch.zeros_like(Ks)
        for b in range(B):
            a, e = int(lo[b]), int(lo[b]) + int(ln[b])
            Ks[b, :, :e - a] = inp.K[b, :, a:e]
            Vs[b, :, :e - a] = inp.V[b, :, a:e]
        be = sharding.CudaBackend()
        stats.append(be.stats(inp.q, Ks, ln, Hkv, S))
        shards.append((be, Vs, ln, lo))
    stats_all = torch.stack(stats, 0)
    total = torch.zeros(B, H, d, dtype=torch.float32, device="cuda")
    for r, (be, Vs, ln, lo) in enumerate(shards):
        part, idx = be.sample_gather(stats_all, r, R, lo, Vs, ln, S, "stratified", 8, 1, return_idx=True)
        total += part
        owner += (idx >= 0).int()
        merged = torch.where(idx >= 0, idx, merged)
    torch.cuda.synchronize()
    assert torch.all(owner == 1)
    assert (merged != full_idx).float().mean().item() < 2e-3
    assert (total.to(torch.bfloat16).float() - full_out.float()).abs().max().item() < 3e-2
