"""Pins for the S^2ANTA-flash oracle (-m "not gpu"; SURVEY 8(f) NEXT-1, App. N Algs.):
merge exactness against the global partition function and dense attention (S:276, S:756 9a), the
SPEC's trivial merge cases, exact unbiasedness over a0 in closed form, single-tile
flash == global systematic sampling (S:756 9c), per-tile counts, the paper's operating
point S_tile = 2048 / 128 = 16, and the sample-waste effect against prop (9e)."""
import math

import numpy as np

from oracle import santa_oracle as o


def test_tile_budget_rule():
    # P:1907 / P:1937: 32k tokens, tile 256, S = 2048 -> T = 128, S_tile = 16
    assert o.flash_tile_budget(32768, 256, 2048) == 16
    assert o.flash_tile_budget(32768, 256, 256) == 2
    assert o.flash_tile_budget(1000, 256, 100) == 25
    assert o.flash_tile_budget(32768, 256, 1) == 1      # never 0
    assert o.flash_tile_budget(1024, 256, 6) == 2       # 1.5 rounds up
    assert o.flash_tile_budget(1024, 256, 5) == 1       # 1.25 rounds down


def test_merge_exact_partition_function_and_dense():
    """S:756 (9a): exp(m*) Z equals the global sum_n exp(s_n) to 1e-10 relative; merging the EXACT
    tile partials O~_t = S_tile sum_{n in t} (u_n / l_t) V_n gives dense softmax(s) V (Eq. 1)."""
    rng = np.random.default_rng(1)
    for trial in range(50):
        n = int(rng.integers(1, 3000))
        B_tile = int(rng.choice([32, 64, 256]))
        s = rng.normal(scale=3.0, size=n)
        V = rng.normal(size=(n, 8))
        m, l, u = o.prop_tile_stats(s, B_tile)
        W = np.exp(m - m.max()) * l
        Zg = np.exp(s - s.max()).sum() * math.exp(s.max() - m.max())
        assert abs(W.sum() - Zg) <= 1e-10 * Zg
        S_tile = 7
        T = m.shape[0]
        O_t = np.stack([S_tile * (u[t * B_tile:(t + 1) * B_tile, None] * V[t * B_tile:(t + 1) * B_tile]).sum(0) / l[t]
                        for t in range(T)])
        np.testing.assert_allclose(o.flash_merge(m, l, O_t, S_tile), o.softmax(s) @ V, rtol=1e-11, atol=1e-12)


def test_merge_trivial_cases():
    """one tile -> O~ / S_tile; two tiles with identical (m, l, O~) -> O~ / S_tile."""
    Ot = np.array([[3.0, -6.0, 9.0]])
    np.testing.assert_allclose(o.flash_merge([0.7], [2.5], Ot, 3), Ot[0] / 3, rtol=1e-15)
    np.testing.assert_allclose(o.flash_merge([0.7, 0.7], [2.5, 2.5], np.vstack([Ot, Ot]), 3), Ot[0] / 3, rtol=1e-15)


def test_flash_is_unbiased_closed_form():
    """Flash is exactly unbiased: E_a0[O] = softmax(s) V for ANY scores (each tile's systematic draw
    is unbiased for its within-tile mean, the merge weights are the exact tile masses).  E over a0
    on a uniform grid (linearity in each a0_t)."""
    rng = np.random.default_rng(2)
    n, B_tile, d, S_tile = 300, 64, 6, 3
    s = rng.normal(scale=2.0, size=n)
    V = rng.normal(size=(n, d))
    m, l, u = o.prop_tile_stats(s, B_tile)
    T = m.shape[0]
    invd = S_tile / l
    M = 3000
    mean = np.zeros(d)
    for k in range(M):
        c = o.prop_counts(u, B_tile, invd, np.full(T, (k + 0.5) / M))
        O_t = np.zeros((T, d))
        for i in np.nonzero(c)[0]:
            O_t[i // B_tile] += c[i] * V[i]
        mean += o.flash_merge(m, l, O_t, S_tile)
    mean /= M
    np.testing.assert_allclose(mean, o.softmax(s) @ V, atol=4.0 * np.abs(V).max() * B_tile / (M * S_tile))


def test_single_tile_flash_equals_global_systematic():
    """S:756 (9c): B_tile >= n_k -> one tile with S_tile = S and the same rows as the search-route
    systematic sampler with u0 = 1 - a0; the merge then returns the plain mean of the rows."""
    rng = np.random.default_rng(3)
    for trial in range(100):
        n = int(rng.integers(1, 256))
        S = int(rng.integers(1, 100))
        q = rng.normal(size=(1, 1, 16))
        K = rng.normal(size=(1, 1, n, 16))
        V = rng.normal(size=(1, 1, n, 16))
        out, idx, det = o.santa_flash_decode(q, K, V, [n], S, seed=trial, B_tile=256, return_details=True)
        dd = det[(0, 0)]
        assert dd["S_tile"] == S
        F = o.cdf(o.softmax(o.scores(q[0, 0], K[0, 0], 1.0 / math.sqrt(16))))
        J = o.inverse_cdf(F, o.thresholds("systematic", S, np.array([1.0 - dd["a0"][0]])))
        np.testing.assert_array_equal(idx[0, 0], J)
        np.testing.assert_allclose(out[0, 0], V[0, 0][J].mean(0), rtol=1e-12, atol=1e-12)


def test_per_tile_counts_and_one_hot_tile():
    """counts per tile sum to S_tile; one-hot mass inside a tile -> O~ = S_tile V_hot."""
    rng = np.random.default_rng(4)
    for _ in range(1000):
        nt = int(rng.integers(1, 257))
        s = rng.normal(scale=rng.uniform(0.1, 8), size=nt)
        m, l, u = o.prop_tile_stats(s, 256)
        S_tile = int(rng.integers(1, 64))
        c = o.prop_counts(u, 256, S_tile / l, rng.random(1))
        assert int(c.sum()) == S_tile
    s = np.full(64, -1e4)
    s[17] = 0.0
    m, l, u = o.prop_tile_stats(s, 64)
    c = o.prop_counts(u, 64, 5 / l, np.array([0.3]))
    assert c[17] == 5 and c.sum() == 5


def test_sample_waste_prop_beats_flash_on_one_hot_tile():
    """S:279 / S:756 (9e), the paper's 'sample waste': mass concentrated in 1 of T = 16 tiles,
    equal total budget S = T S_tile -> prop's MSE below flash's over 200 seeds (one-sided, the gap
    is many standard errors)."""
    rng = np.random.default_rng(5)
    B_tile, T, d = 64, 16, 16
    n = B_tile * T
    q = rng.normal(size=(1, 1, d))
    K = rng.normal(size=(1, 1, n, d)) * 0.3
    K[0, 0, 5 * B_tile:6 * B_tile] += 2.0 * q[0, 0] / np.linalg.norm(q[0, 0])  # the hot tile
    V = rng.normal(size=(1, 1, n, d))
    exact = o.dense_decode(q, K, V, [n])[0, 0]
    S = 2 * T
    ep, ef = [], []
    for seed in range(200):
        outp, _ = o.santa_prop_decode(q, K, V, [n], S, seed=seed, B_tile=B_tile)
        outf, _ = o.santa_flash_decode(q, K, V, [n], S, seed=seed, B_tile=B_tile)
        ep.append(((outp[0, 0] - exact) ** 2).sum())
        ef.append(((outf[0, 0] - exact) ** 2).sum())
    ep, ef = np.array(ep), np.array(ef)
    diff = ef - ep
    assert diff.mean() > 3 * diff.std(ddof=1) / math.sqrt(diff.size)
