"""Pins for the three samplers and the batched decode oracle (-m "not gpu"):
brute-force exact laws at n_k <= 8, closed-form variances, the systematic floor/ceil
invariant, the P:1631 count formula, one-hot exactness, and unbiasedness at 3 sigma."""
import itertools
import math

import numpy as np
import pytest

from oracle import santa_oracle as o

import santa_inputs as si


def _profile(rng, n, zeros=True):
    p = rng.dirichlet(np.ones(n) * 0.7)
    if zeros:
        p = p * (rng.random(n) > 0.25)
        if p.sum() == 0:
            p[0] = 1.0
    return p / p.sum()


def test_iid_brute_force_multinomial_law():
    """n_k = 4, S = 2: oracle tuple frequencies over 2e4 seeds vs the exact law
    P(i1, i2) = p_i1 p_i2 over all n_k^S ordered tuples (chi-square)."""
    p = np.array([0.1, 0.2, 0.3, 0.4])
    F = o.cdf(p)
    S, N = 2, 20000
    counts = {}
    for s in range(N):
        u = o.sampler_uniforms("iid", S, s, 0, 0, 0)
        t = tuple(o.inverse_cdf(F, o.thresholds("iid", S, u)))
        counts[t] = counts.get(t, 0) + 1
    chi2 = 0.0
    for t in itertools.product(range(4), repeat=S):
        e = N * np.prod(p[list(t)])
        chi2 += (counts.get(t, 0) - e) ** 2 / e
    assert chi2 < 45.0          # 15 dof; p ~ 1e-4


def test_stratified_exact_law_by_enumeration():
    """P(J_m = j) = S |[F(j-1),F(j)) cap I_m| -- checked by enumerating the
    stratum's threshold over a fine deterministic grid u in [0,1)."""
    rng = np.random.default_rng(0)
    for _ in range(30):
        n, S = int(rng.integers(2, 9)), int(rng.integers(1, 6))
        p = _profile(rng, n)
        F = o.cdf(p)
        law = o.stratum_law(p, S)
        grid = (np.arange(4000) + 0.5) / 4000
        Tg = np.stack([o.thresholds("stratified", S, np.full(S, g)) for g in grid])  # [grid, S]
        for m in range(S):
            J = o.inverse_cdf(F, Tg[:, m])
            freq = np.bincount(J, minlength=n) / grid.size
            np.testing.assert_allclose(freq, law[m], atol=1e-3)
        # the law reproduces the paper's unbiasedness: (1/S) sum_m E[V_Jm] = sum p_j V_j
        np.testing.assert_allclose(law.sum(0) / S, p, atol=1e-12)


def test_stratified_spec_examples():
    for s in range(50):
        u = o.sampler_uniforms("stratified", 2, s, 0, 0, 0)
        assert sorted(o.inverse_cdf(o.cdf([0.5, 0.5]), o.thresholds("stratified", 2, u))) == [0, 1]
        u = o.sampler_uniforms("stratified", 4, s, 0, 0, 0)
        assert sorted(o.inverse_cdf(o.cdf([0.25] * 4), o.thresholds("stratified", 4, u))) == [0, 1, 2, 3]


def test_systematic_floor_ceil_invariant_and_count_formula():
    """Every systematic count c_j is floor(S p_j) or ceil(S p_j), sum = S (north star);
    the per-key count form of Alg. prop-pass2 gives the same counts."""
    rng = np.random.default_rng(1)
    for trial in range(300):
        n, S = int(rng.integers(1, 40)), int(rng.integers(1, 70))
        p = _profile(rng, n)
        F = o.cdf(p)
        u = o.sampler_uniforms("systematic", S, trial, 0, 0, 0)
        J = o.inverse_cdf(F, o.thresholds("systematic", S, u))
        c = np.bincount(J, minlength=n)
        assert c.sum() == S
        assert np.all(c >= np.floor(S * p - 1e-9)) and np.all(c <= np.ceil(S * p + 1e-9))
        np.testing.assert_array_equal(o.systematic_counts_formula(F, S, float(u[0])), c)


def test_systematic_spec_examples():
    for s in range(200):
        u = o.sampler_uniforms("systematic", 10, s, 0, 0, 0)
        J = o.inverse_cdf(o.cdf([0.1, 0.9]), o.thresholds("systematic", 10, u))
        assert (J == 0).sum() == 1
        u = o.sampler_uniforms("systematic", 2, s, 0, 0, 0)
        assert sorted(o.inverse_cdf(o.cdf([0.5, 0.5]), o.thresholds("systematic", 2, u))) == [0, 1]


def test_systematic_exact_law_is_unbiased_and_matches_brute_force():
    """The breakpoint sweep's exact mean equals AV (Prop. P:673-705), and its variance
    equals a brute-force average over a fine grid of u."""
    rng = np.random.default_rng(2)
    for _ in range(40):
        n, S, d = int(rng.integers(2, 9)), int(rng.integers(1, 9)), 3
        p = _profile(rng, n)
        V = rng.normal(size=(n, d))
        mean, var = o.systematic_law(p, V, S)
        np.testing.assert_allclose(mean, p @ V, atol=1e-12)
        F = o.cdf(p)
        grid = (np.arange(40000) + 0.5) / 40000
        outs = np.stack([V[o.inverse_cdf(F, (np.arange(S) + u) / S)].mean(0) for u in grid[::10]])
        np.testing.assert_allclose(outs.var(0), var, atol=2e-3)


def test_variance_closed_forms_and_dominance():
    """iid VarTrace = tr(Sigma)/S against brute force over all n^S tuples;
    stratified (1/S^2) sum_m tr(Sigma_m) <= iid (Thm P:710-751)."""
    rng = np.random.default_rng(3)
    for _ in range(50):
        n, S, d = int(rng.integers(2, 6)), int(rng.integers(1, 4)), 2
        p = _profile(rng, n, zeros=False)
        V = rng.normal(size=(n, d))
        mu = p @ V
        brute = 0.0
        for t in itertools.product(range(n), repeat=S):
            w = np.prod(p[list(t)])
            brute += w * np.sum((V[list(t)].mean(0) - mu) ** 2)
        assert abs(o.var_trace_iid(p, V, S) - brute) < 1e-12
        assert abs(o.var_iid_per_coord(p, V, S).sum() - brute) < 1e-12
        _, vs = o.var_stratified(p, V, S)
        assert vs <= o.var_trace_iid(p, V, S) + 1e-12
    # SPEC analysis examples
    assert abs(o.var_trace_iid([0.5, 0.5], np.array([[1.0], [-1.0]]), 4) - 0.25) < 1e-15
    assert o.var_stratified([0.5, 0.5], np.array([[1.0], [-1.0]]), 2)[1] == 0.0


def test_one_hot_attention_is_exact_all_modes():
    """One-hot attention (logit margin >= 1e4) -> out = V_j exactly for every mode and S."""
    inp = si.make_decode_inputs(1, 4, 2, 16, 37, dtype="bf16", seed=3)
    q = inp.q.clone()
    K = inp.K.clone()
    hot = 11
    K[:, :, hot, :] = 0
    K[:, :, hot, 0] = 100.0
    q[:, :, 0] = 100.0
    for mode in o.MODES:
        for S in (1, 3, 64):
            out, idx = o.santa_decode(si.as_bits(q), si.as_bits(K), si.as_bits(inp.V),
                                      [37], S, mode, seed=9)
            assert np.all(idx == hot)
            V = o.to_f64(si.as_bits(inp.V))
            for h in range(4):
                np.testing.assert_array_equal(out[0, h], V[0, h // 2, hot])


@pytest.mark.parametrize("mode", o.MODES)
def test_unbiasedness_3sigma(mode):
    """Mean over 1e4 seeds converges to dense AV within 3 sigma (Props), with
    sigma from the exact variance of each scheme (iid closed form; stratified closed
    form; systematic exact breakpoint law).  Family-wise rule of reading #17."""
    rng = np.random.default_rng(4)
    n, d, S, N = 24, 6, 4, 10000
    s = rng.normal(size=n) * 1.5
    p = o.softmax(s)
    V = rng.normal(size=(n, d))
    F = o.cdf(p)
    outs = np.empty((N, d))
    for seed in range(N):
        u = o.sampler_uniforms(mode, S, seed, 0, 0, 0)
        outs[seed] = o.gather_mean(V, o.inverse_cdf(F, o.thresholds(mode, S, u)))
    if mode == "iid":
        var = o.var_iid_per_coord(p, V, S)
    elif mode == "stratified":
        var = o.var_stratified(p, V, S)[0]
    else:
        var = o.systematic_law(p, V, S)[1]
    z = (outs.mean(0) - p @ V) / np.sqrt(var / N)
    assert np.max(np.abs(z)) < 3.6          # Sidak-adjusted 3 sigma for d = 6 coordinates
    # and the empirical variance matches the exact variance (5%)
    np.testing.assert_allclose(outs.var(0), var, rtol=0.06)


def test_santa_decode_batched_matches_single_query_path():
    """The batched (b, h) loop with GQA (k(h) = floor(h/G)) and ragged seqlens
    equals the single-query santa_estimate on the sliced rows."""
    inp = si.make_decode_inputs(2, 4, 2, 8, [13, 5], dtype="bf16", seed=1)
    out, idx = o.santa_decode(si.as_bits(inp.q), si.as_bits(inp.K), si.as_bits(inp.V),
                              [13, 5], 6, "stratified", seed=3, offset=2)
    q, K, V = (o.to_f64(si.as_bits(t)) for t in (inp.q, inp.K, inp.V))
    for b, n in enumerate([13, 5]):
        for h in range(4):
            u = o.sampler_uniforms("stratified", 6, 3, 2, h, b)
            e, j = o.santa_estimate(q[b, h], K[b, h // 2, :n], V[b, h // 2, :n],
                                    1 / math.sqrt(8), 6, "stratified", u)
            np.testing.assert_array_equal(idx[b, h], j)
            np.testing.assert_array_equal(out[b, h], e)
            assert np.all(j < n)


def test_sequence_sharding_equals_unsharded():
    """Reading #18: with contiguous shards and global thresholds, the sharded sampler
    returns exactly the unsharded indices (stratified and systematic; iid too)."""
    rng = np.random.default_rng(5)
    for trial in range(40):
        n, S, R = int(rng.integers(5, 300)), int(rng.integers(1, 64)), int(rng.integers(1, 6))
        s = rng.normal(size=n) * rng.choice([0.5, 3.0, 8.0])
        for mode in o.MODES:
            u = o.sampler_uniforms(mode, S, trial, 0, 0, 0)
            T = o.thresholds(mode, S, u)
            J = o.inverse_cdf(o.cdf(o.softmax(s)), T)
            bounds = o.shard_bounds(n, R)
            stats = [o.shard_stats(s[a:b]) for a, b in bounds]
            got = np.full(S, -1)
            for r, (a, b) in enumerate(bounds):
                mine, ids = o.shard_sample(s[a:b], a, stats, r, T)
                assert np.all(got[mine] == -1)
                got[mine] = ids
            diff = np.nonzero(got != J)[0]
            F = o.cdf(o.softmax(s))
            for m in diff:  # only exact-boundary rounding cases may differ
                lo, hi = min(got[m], J[m]), max(got[m], J[m])
                assert got[m] >= 0 and np.all(np.abs(F[lo:hi] - T[m]) < 1e-12)
