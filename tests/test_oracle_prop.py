"""Pins for the S^2ANTA-prop oracle (-m "not gpu"; SURVEY 8(f) NEXT-2, App. M Algs.):
the SPEC's worked largest-remainder example, brute-force optimality of the
largest-remainder allocation, budget conservation on 10^4 random allocations (S:756 9b),
single-tile prop == global systematic sampling (S:756 9c), the per-tile count law of
Kernel 3 in closed form, exact unbiasedness when every quota is an integer, and the
large-budget error against the iid closed form (S:756 9d)."""
import itertools
import math

import numpy as np

from conftest import golden
from oracle import santa_oracle as o


def _paper_value(key):
    for line in open(golden("paper_values.txt")):
        line = line.split("#")[0]
        if "=" in line and line.split("=")[0].strip() == key:
            return line.split("=", 1)[1].strip()
    raise KeyError(key)


def test_largest_remainder_worked_example():
    """W proportional to [0.55, 0.30, 0.15], S = 10 -> quotas [5.5, 3.0, 1.5], floors
    [5, 3, 1], one remainder; fractional parts 0.5 tie between tiles 0 and 2 -> lower index."""
    lhs, rhs = _paper_value("prop_lr_example").split("->")
    W = np.array([float(x) for x in lhs.split()[0].split("=")[1].split(",")])
    S = int(lhs.split()[1].split("=")[1])
    want = [int(x) for x in rhs.split()]
    # through the whole budget kernel: m_t = 0 for every tile, l_t = W_t
    St, invd, q = o.prop_budgets(np.zeros(3), W, S)
    assert St.tolist() == want
    np.testing.assert_allclose(q, [5.5, 3.0, 1.5], rtol=1e-15)
    np.testing.assert_allclose(invd, np.array(want) / W, rtol=1e-15)


def test_largest_remainder_is_the_lexicographic_least_squares_allocation():
    """Brute force over every composition of S into T non-negative parts (T <= 4, S <= 7): the
    largest-remainder allocation minimises sum_t (S_t - q_t)^2, and among the minimisers (equal
    fractional parts) it is the lexicographically greatest (extra samples to lower tiles)."""
    rng = np.random.default_rng(5)
    for trial in range(300):
        T = int(rng.integers(1, 5))
        S = int(rng.integers(1, 8))
        if trial % 3 == 0:  # force ties: quotas on a coarse grid
            W = rng.integers(1, 4, size=T).astype(np.float64)
        else:
            W = rng.random(T) + 1e-3
        q = S * W / W.sum()
        best, best_key = None, None
        for comp in itertools.product(range(S + 1), repeat=T):
            if sum(comp) != S:
                continue
            err = round(float(sum((c - x) ** 2 for c, x in zip(comp, q))), 9)
            key = (err, tuple(-c for c in comp))
            if best_key is None or key < best_key:
                best, best_key = comp, key
        assert tuple(o.largest_remainder(q, S).tolist()) == best, (W, S)


def test_budget_conservation_random_allocations():
    """S:756 (9b): sum_t S_t = S on 10^4 random allocations; every S_t in {floor q_t, ceil q_t};
    invdelta_t = 0 exactly where S_t = 0."""
    rng = np.random.default_rng(11)
    for _ in range(10000):
        T = int(rng.integers(1, 40))
        S = int(rng.integers(1, 600))
        m = rng.normal(scale=3.0, size=T)
        l = rng.random(T) * 64 + 1.0
        St, invd, q = o.prop_budgets(m, l, S)
        assert int(St.sum()) == S
        assert np.all(St >= np.floor(q)) and np.all(St <= np.floor(q) + 1)
        assert np.all((invd == 0) == (St == 0))


def test_single_tile_prop_equals_global_systematic():
    """S:756 (9c): with one tile (B_tile >= n_k) the budget is S, invdelta = S / l and Kernel 3's
    counts select the same rows as the search-route systematic sampler J_m = min{j : F(j) > T_m},
    T_m = (m + u0)/S, with u0 = 1 - a0 (reading #9)."""
    rng = np.random.default_rng(3)
    for trial in range(200):
        n = int(rng.integers(1, 300))
        S = int(rng.integers(1, 200))
        s = rng.normal(scale=2.0, size=n)
        m, l, u = o.prop_tile_stats(s, n + int(rng.integers(0, 5)))
        St, invd, _ = o.prop_budgets(m, l, S)
        assert St.tolist() == [S]
        a0 = o.philox_uniforms(trial, 0, o.TAG_PROP_TILE_OFFSET, 0, 0, np.arange(1))
        J_prop = np.repeat(np.arange(n), o.prop_counts(u, n, invd, a0))
        F = o.cdf(o.softmax(s))
        J_sys = o.inverse_cdf(F, o.thresholds("systematic", S, np.array([1.0 - a0[0]])))
        np.testing.assert_array_equal(J_prop, J_sys)


def test_kernel3_count_law_closed_form():
    """Per tile, the counts are systematic resampling of u / l_t with S_t draws: sum_n c_n = S_t,
    c_n in {floor(S_t u_n / l_t), ceil(...)} up to the running sum's rounding, and over a0 on a
    uniform grid of M points the mean count equals S_t u_n / l_t within 1/M."""
    rng = np.random.default_rng(8)
    s = rng.normal(scale=1.5, size=200)
    B_tile = 48
    m, l, u = o.prop_tile_stats(s, B_tile)
    St, invd, q = o.prop_budgets(m, l, 97)
    T = m.shape[0]
    # quotas are S times each tile's share of the softmax mass (P:1607-1608 vs Eq. 1)
    pt = np.add.reduceat(o.softmax(s), np.arange(0, 200, B_tile))
    np.testing.assert_allclose(q, 97 * pt, rtol=1e-12)
    M = 400
    mean = np.zeros(200)
    for k in range(M):
        c = o.prop_counts(u, B_tile, invd, np.full(T, (k + 0.5) / M))
        for t in range(T):
            assert int(c[t * B_tile:(t + 1) * B_tile].sum()) == St[t]
        mean += c
    mean /= M
    tile = np.arange(200) // B_tile
    expect = St[tile] * u / l[tile]
    np.testing.assert_allclose(mean, expect, atol=1.0 / M + 1e-12)
    c = o.prop_counts(u, B_tile, invd, np.full(T, 0.37))
    assert np.all(c >= np.floor(expect - 1e-9)) and np.all(c <= np.ceil(expect + 1e-9))


def test_integer_quotas_are_unbiased_against_dense_attention():
    """When every quota q_t = S W_t / Z is an integer (T tiles holding permutations of the same
    scores, S a multiple of T) the largest-remainder rounding is void and E_a0[out] is exactly the
    dense softmax(s) V (Eq. 1).  E over a0 by a uniform grid (linearity in each a0_t)."""
    rng = np.random.default_rng(21)
    B_tile, T, d, S = 16, 4, 8, 12
    base = rng.normal(scale=1.2, size=B_tile)
    s = np.concatenate([rng.permutation(base) for _ in range(T)])
    V = rng.normal(size=(B_tile * T, d))
    m, l, u = o.prop_tile_stats(s, B_tile)
    St, invd, q = o.prop_budgets(m, l, S)
    assert St.tolist() == [S // T] * T
    M = 2000
    mean = np.zeros(d)
    for k in range(M):
        c = o.prop_counts(u, B_tile, invd, np.full(T, (k + 0.5) / M))
        mean += (c[:, None] * V).sum(0) / S
    mean /= M
    exact = o.softmax(s) @ V
    np.testing.assert_allclose(mean, exact, atol=2.0 * np.abs(V).max() * (B_tile * T) / (M * S))


def test_decode_batched_consistency_and_large_budget():
    """santa_prop_decode over a GQA batch: emitted rows per tile equal the budgets, out equals the
    gather-mean of its own rows (Eq. 4), and S:756 (9d): S = 4096 on n_k = 1024 gives a
    relative error well below the iid estimator's."""
    rng = np.random.default_rng(4)
    B, H, Hkv, d, n = 2, 4, 2, 16, 300
    q = rng.normal(size=(B, H, d))
    K = rng.normal(size=(B, Hkv, n, d))
    V = rng.normal(size=(B, Hkv, n, d))
    seqlens = np.array([300, 131])
    out, idx, det = o.santa_prop_decode(q, K, V, seqlens, 40, seed=9, B_tile=64, return_details=True)
    for (b, h), dd in det.items():
        n_b = seqlens[b]
        tiles = idx[b, h] // 64
        assert np.bincount(tiles, minlength=dd["St"].shape[0]).tolist() == dd["St"].tolist()
        assert np.all(np.diff(idx[b, h]) >= 0) and idx[b, h].max() < n_b
    np.testing.assert_allclose(out, o.out_given_idx(V, idx), rtol=1e-13, atol=1e-13)

    # S:756 (9d) asks for a small error at S = 4096, n_k = 1024; its 0.05 figure assumes a score
    # distribution it does not state, so the pin here is the closed form instead: prop is systematic
    # within tiles, so its error stays below half the iid estimator's exact RMS error
    # sqrt(tr Cov / S) / ||out|| (Prop. A.1, var_trace_iid) on every seed
    S, nk = 4096, 1024
    for seed in range(5):
        r = np.random.default_rng(100 + seed)
        q1 = r.normal(size=(1, 1, 32))
        K1 = r.normal(size=(1, 1, nk, 32))
        V1 = r.normal(size=(1, 1, nk, 32))
        est, _ = o.santa_prop_decode(q1, K1, V1, [nk], S, seed=seed, B_tile=64)
        exact = o.dense_decode(q1, K1, V1, [nk])
        p = o.softmax(o.scores(q1[0, 0], K1[0, 0], 1.0 / math.sqrt(32)))
        iid_rms = math.sqrt(o.var_trace_iid(p, V1[0, 0], S)) / np.linalg.norm(exact)
        assert o.fidelity(est, exact)[0] < 0.5 * iid_rms
