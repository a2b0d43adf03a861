"""Shared helpers for the -m gpu parity tests: run the CUDA path through the C-ABI binding
and compare with the oracle on the same seeded inputs."""
import numpy as np
import torch

import paper_2605_01910_b200 as santa
import santa_inputs as si
from oracle import santa_oracle as o

TOL = {"bf16": 2e-2, "f16": 2e-2, "f32": 1e-5}   # north star: output parity given identical indices


def to_cuda(inp):
    dev = "cuda"
    inp.q = inp.q.to(dev)
    inp.K = inp.K.to(dev)
    inp.V = inp.V.to(dev)
    inp.seqlens = inp.seqlens.to(dev)
    if inp.K_pool is not None:
        inp.K_pool = inp.K_pool.to(dev)
        inp.V_pool = inp.V_pool.to(dev)
        inp.page_table = inp.page_table.to(dev)
    if inp.Kt is not None:
        inp.Kt = inp.Kt.to(dev)
    return inp


def gpu_decode(inp, S, mode, seed, offset=0, paged=False, max_seqlen=None, head_offset=0, batch_offset=0,
               path="auto"):
    """path: "auto" (what santa_decode_attention runs), "step" (force the single pipelined launch)
    or "two_kernel" (score pass + sampler kernel)."""
    if paged:
        out, idx = santa.decode(inp.q, inp.K_pool, inp.V_pool, inp.seqlens, S, mode, seed, offset,
                                n_kv_heads=inp.n_kv_heads, page_table=inp.page_table, page_size=inp.page_size,
                                max_seqlen=max_seqlen or inp.max_seqlen, return_idx=True,
                                head_offset=head_offset, batch_offset=batch_offset, path=path)
    else:
        out, idx = santa.decode(inp.q, inp.K, inp.V, inp.seqlens, S, mode, seed, offset,
                                max_seqlen=max_seqlen, return_idx=True, head_offset=head_offset,
                                batch_offset=batch_offset, path=path)
    torch.cuda.synchronize()
    return out, idx


def oracle_decode(inp, S, mode, seed, offset=0, head_offset=0, batch_offset=0):
    q, K, V = si.as_bits(inp.q), si.as_bits(inp.K), si.as_bits(inp.V)
    return o.santa_decode(q, K, V, inp.seqlens.cpu().numpy(), S, mode, seed, offset,
                          head_offset=head_offset, batch_offset=batch_offset, return_details=True)


def check_parity(inp, out_gpu, idx_gpu, S, mode, seed, offset=0, head_offset=0, batch_offset=0,
                 max_mismatch_rate=5e-3):
    """Index parity with the 1e-6 boundary exemption (reading #19) and output parity on the
    GPU's own indices (reading #16).  Returns (total, mismatches, exempt)."""
    out_o, idx_o, det = oracle_decode(inp, S, mode, seed, offset, head_offset, batch_offset)
    idx_g = idx_gpu.cpu().numpy().astype(np.int64)
    total, mism, exempt, fails = o.index_mismatch_report(det["F"], det["T"], idx_o, idx_g)
    assert not fails, f"non-exempt index mismatches: {fails[:5]} (of {len(fails)})"
    assert mism <= max_mismatch_rate * total, (mism, total)
    ref = o.out_given_idx(si.as_bits(inp.V), idx_g)
    got = out_gpu.float().cpu().numpy().astype(np.float64)
    err = np.abs(got - ref).max()
    assert err <= TOL[inp.dtype], f"output max-abs err {err} > {TOL[inp.dtype]}"
    return total, mism, exempt


# ---- S^2ANTA-prop / -flash row parity (readings #25, #26) --------------------------------------
# The tile estimators decide rows by comparing the tile's uniform a0 with count boundaries:
# row j of tile t is min{n : a0 + U_n S_t / l_t >= j}, i.e. the in-tile threshold
# tau_j = (j - a0) / S_t against the tile CDF U_n / l_t.  The north-star rule ("a uniform within
# 1e-6 of a CDF boundary") carried to the tile, in the same units as the exact path's rule (CDF
# units, where T_m = (m + u_m) / S is compared with F): a GPU/oracle row mismatch is exempt iff
# every crossed tile-CDF boundary U_n / l_t lies within ROW_TOL of tau_j, i.e. |y - j| <= ROW_TOL * S_t
# with y = a0 + U_n S_t / l_t (reading #25; "1e-6 in tile-CDF units").
ROW_TOL = 1e-6


def lr_valid(Sg, q, S, tol):
    """Sg is a largest-remainder allocation of quotas within tol of q: sum = S, every S_t within
    1 + tol of q_t, and no tile rounded down keeps a larger remainder than a tile rounded up."""
    if int(Sg.sum()) != S or np.any(np.abs(Sg - q) >= 1 + tol):
        return False
    up = Sg > q
    down_rem = (q - Sg)[~up]
    up_rem = (1.0 - (Sg - q))[up]
    if down_rem.size == 0 or up_rem.size == 0:
        return True
    return down_rem.max() <= up_rem.min() + 2 * tol


def _row_boundaries_near(dd, t, B_tile, n, St_t, lo, hi, j):
    u = dd["u"][t * B_tile:min((t + 1) * B_tile, n)]
    y = dd["a0"][t] + np.cumsum(u)[lo - t * B_tile:hi - t * B_tile] * (St_t / dd["l"][t])
    return bool(np.all(np.abs(y - j) <= ROW_TOL * St_t)), (y - j) / St_t


def prop_parity(inp, out_g, idx_g, S, seed, offset=0, head_offset=0, batch_offset=0, B_tile=64):
    """S^2ANTA-prop GPU rows vs santa_prop_decode.  Budgets: a head whose GPU budgets differ from
    the oracle's must be a valid largest-remainder allocation of the ORACLE's quotas within
    1e-6 * S (the 1e-6 CDF-unit rule in quota units: q_t = S W_t / Z) -- such heads are counted and
    returned.  Rows: compared tile by tile wherever the two budgets agree (every tile of every
    head), mismatches only under ROW_TOL.  Output: on the GPU's own rows (reading #16).
    Returns (heads, heads with different budgets, rows compared, row mismatches, exempt)."""
    q, K, V = si.as_bits(inp.q), si.as_bits(inp.K), si.as_bits(inp.V)
    seqlens = inp.seqlens.cpu().numpy()
    _, idx_o, det = o.santa_prop_decode(q, K, V, seqlens, S, seed, offset, B_tile=B_tile,
                                        head_offset=head_offset, batch_offset=batch_offset, return_details=True)
    idx_g = idx_g.cpu().numpy().astype(np.int64)
    heads = budget_diff = compared = mism = exempt = 0
    for (b, h), dd in det.items():
        heads += 1
        n = int(seqlens[b])
        ig, io = idx_g[b, h], idx_o[b, h]
        assert ig.min() >= 0 and ig.max() < n and np.all(np.diff(ig) >= 0), (b, h)
        St = dd["St"]
        T = St.shape[0]
        Sg = np.bincount(ig // B_tile, minlength=T)
        assert Sg.shape[0] == T
        if not np.array_equal(Sg, St):
            budget_diff += 1
            assert lr_valid(Sg, dd["q"], S, 1e-6 * S + 1e-12), (b, h, np.nonzero(Sg != St))
        offo = np.concatenate([[0], np.cumsum(St)])
        offg = np.concatenate([[0], np.cumsum(Sg)])
        for t in np.nonzero((St == Sg) & (St > 0))[0]:
            ro, rg = io[offo[t]:offo[t + 1]], ig[offg[t]:offg[t + 1]]
            compared += int(St[t])
            for k in np.nonzero(ro != rg)[0]:
                ok, dy = _row_boundaries_near(dd, t, B_tile, n, St[t], min(ro[k], rg[k]), max(ro[k], rg[k]), k + 1)
                assert ok, (b, h, int(t), int(k), int(ro[k]), int(rg[k]), dy)
                exempt += 1
            mism += int((ro != rg).sum())
    ref = o.out_given_idx(V, idx_g)
    got = out_g.float().cpu().numpy().astype(np.float64)
    err = np.abs(got - ref).max()
    assert err <= TOL[inp.dtype], f"output max-abs err {err} > {TOL[inp.dtype]}"
    return heads, budget_diff, compared, mism, exempt


def flash_parity(inp, out_g, idx_g, S, tile_len, seed, offset=0, head_offset=0, batch_offset=0):
    """S^2ANTA-flash GPU rows vs santa_flash_decode: budgets are fixed by (n, tile_len, S), rows
    must agree one by one except under ROW_TOL, and the output must equal the oracle's merge
    (fp64 W_t, Z) of the GPU's own rows.  Returns (rows compared, row mismatches)."""
    q, K, V = si.as_bits(inp.q), si.as_bits(inp.K), si.as_bits(inp.V)
    seqlens = inp.seqlens.cpu().numpy()
    _, idx_o, det = o.santa_flash_decode(q, K, V, seqlens, S, seed, offset, B_tile=tile_len,
                                         head_offset=head_offset, batch_offset=batch_offset, return_details=True)
    idx_g = idx_g.cpu().numpy().astype(np.int64)
    Vf = o.to_f64(V)
    G = inp.q.shape[1] // V.shape[1]
    got = out_g.float().cpu().numpy().astype(np.float64)
    compared = mism = 0
    for (b, h), dd in det.items():
        n = int(seqlens[b])
        St, T = dd["S_tile"], dd["m"].shape[0]
        M = St * T
        ig = idx_g[b, h]
        assert np.all(ig[M:] == -1), (b, h)
        ig = ig[:M]
        io = idx_o[b, h, :M]
        assert ig.min() >= 0 and ig.max() < n and np.all(np.diff(ig) >= 0), (b, h)
        assert np.array_equal(np.bincount(ig // tile_len, minlength=T), np.full(T, St)), (b, h)
        for m in np.nonzero(io != ig)[0]:
            t, j = m // St, m % St + 1
            ok, dy = _row_boundaries_near(dd, t, tile_len, n, St, min(io[m], ig[m]), max(io[m], ig[m]), j)
            assert ok, (b, h, int(m), int(io[m]), int(ig[m]), dy)
        mism += int((io != ig).sum())
        compared += M
        Vb = Vf[b, h // G, :n]
        O_t = np.zeros((T, Vb.shape[1]))
        for r in ig:
            O_t[r // tile_len] += Vb[r]
        ref = o.flash_merge(dd["m"], dd["l"], O_t, St)
        err = np.abs(got[b, h] - ref).max()
        assert err <= TOL[inp.dtype], f"({b},{h}) output max-abs err {err} > {TOL[inp.dtype]}"
    assert mism <= 5e-3 * compared, (mism, compared)
    return compared, mism
