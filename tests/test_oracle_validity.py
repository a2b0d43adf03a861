"""Pins (-m "not gpu") for the oracle's validity machinery -- the parts every GPU parity verdict
rests on ("What's weak" #1):

* ``index_mismatch_report``: the north-star exemption rule (reading #19) on hand-built
  CDFs whose verdicts are worked out by hand below (boundary at 5e-7 exempt, at 2e-6 not, a
  two-index gap with one far boundary not, both boundaries near exempt, out-of-range indices
  never exempt, the lo/hi slice edges);
* ``santa_from_scores`` (the config-5 value stage on GIVEN scores): composed with the
  exact score stage it must reproduce ``santa_decode`` (pinned independently in
  test_oracle_core / test_oracle_samplers) index for index, and one-hot scores give V_j exactly;
* the PER-HEAD branch of ``bernoulli_scores`` (Eq. 5, Philox tag 2 keyed by the global
  query head, reading #1): equal to ``bernoulli_qk_head`` per head with the stream drawn from the
  KAT-pinned ``philox_uniforms``, and exact when every |q_i| equals the norm.
"""
import math

import numpy as np
import pytest

import santa_inputs as si
from oracle import santa_oracle as o


# ---------------------------------------------------------------------------------------------
# index_mismatch_report (reading #19)
# ---------------------------------------------------------------------------------------------

F4 = np.array([0.1, 0.3, 0.6, 1.0])


def _report(F, T, jo, jg, tol=1e-6):
    idx_o = np.array(jo, dtype=np.int64).reshape(1, 1, -1)
    idx_g = np.array(jg, dtype=np.int64).reshape(1, 1, -1)
    return o.index_mismatch_report({(0, 0): np.asarray(F)}, {(0, 0): np.asarray(T, dtype=np.float64)}, idx_o, idx_g,
                                   tol)


def test_exemption_boundary_within_tolerance():
    # T = 0.3 + 5e-7: J = min{j : F(j) > T} = 2; a GPU index 1 differs only across the
    # boundary F(1) = 0.3, which is 5e-7 < 1e-6 from T -> exempt
    T = [0.3 + 5e-7]
    assert o.inverse_cdf(F4, np.array(T))[0] == 2
    assert _report(F4, T, [2], [1]) == (1, 1, 1, [])


def test_exemption_boundary_outside_tolerance():
    T = [0.3 + 2e-6]          # 2e-6 from the only boundary crossed -> a failure
    tot, mism, ex, fails = _report(F4, T, [2], [1])
    assert (tot, mism, ex) == (1, 1, 0) and fails == [(0, 0, 0, 2, 1, T[0])]


def test_exemption_two_index_gap():
    T = [0.3 + 5e-7]
    # GPU 0 vs oracle 2 crosses F(0) = 0.1 (far) and F(1) = 0.3 (near): every boundary must be near
    tot, mism, ex, fails = _report(F4, T, [2], [0])
    assert (mism, ex, len(fails)) == (1, 0, 1)
    # a cluster of boundaries all within 1e-6 of T: exempt even two atoms apart
    F = np.array([0.3, 0.3 + 1e-7, 0.6, 1.0])
    assert o.inverse_cdf(F, np.array(T))[0] == 2
    assert _report(F, T, [2], [0])[:3] == (1, 1, 1)
    # the same cluster, GPU on the other side: oracle 2, GPU 3 crosses F(2) = 0.6 -> failure
    assert _report(F, T, [2], [3])[2] == 0


def test_exemption_slice_edges_and_range():
    # last boundary: T = 1 - 4e-7 against F(2) = 1 - 1e-7 ... the crossing at j = 2 is near
    F = np.array([0.2, 0.5, 1.0 - 1e-7, 1.0])
    T = [1.0 - 4e-7]
    assert o.inverse_cdf(F, np.array(T))[0] == 2
    assert _report(F, T, [2], [3])[2] == 1           # crosses F(2) only (slice [2:3])
    # the slice is [min, max): the boundary AT the larger index is not crossed
    T2 = [0.5 + 3e-7]                                 # oracle 2; GPU 1 crosses F(1) = 0.5 only
    assert _report(F, T2, [2], [1])[2] == 1
    # indices outside [0, n] are never exempt (a GPU index past the sequence or negative)
    assert _report(F, T, [2], [5])[2] == 0
    assert _report(F, T, [2], [-1])[2] == 0
    # equal indices are not mismatches; totals count every (b, h, m)
    tot, mism, ex, fails = _report(F4, [0.05, 0.2, 0.7], [0, 1, 3], [0, 1, 3])
    assert (tot, mism, ex, fails) == (3, 0, 0, [])


def test_exemption_tolerance_argument():
    T = [0.3 + 5e-7]
    assert _report(F4, T, [2], [1], tol=1e-7)[2] == 0
    assert _report(F4, T, [2], [1], tol=1e-6)[2] == 1


def test_exemption_multi_head_bookkeeping():
    """Per-(b, h) CDFs are looked up by key; failures report (b, h, m, j_oracle, j_gpu, T)."""
    F = {(0, 0): F4, (0, 1): np.array([0.5, 1.0]), (1, 0): F4, (1, 1): np.array([0.5, 1.0])}
    T = {(0, 0): np.array([0.3 + 5e-7, 0.9]), (0, 1): np.array([0.5 + 1e-8, 0.2]),
         (1, 0): np.array([0.05, 0.65]), (1, 1): np.array([0.7, 0.5 + 3e-6])}
    io = np.array([[[2, 3], [1, 0]], [[0, 3], [1, 1]]])
    ig = np.array([[[1, 3], [0, 0]], [[0, 3], [1, 0]]])
    tot, mism, ex, fails = o.index_mismatch_report(F, T, io, ig)
    assert (tot, mism, ex) == (8, 3, 2)
    assert fails == [(1, 1, 1, 1, 0, float(T[(1, 1)][1]))]


# ---------------------------------------------------------------------------------------------
# santa_from_scores
# ---------------------------------------------------------------------------------------------

@pytest.mark.parametrize("mode", o.MODES)
def test_from_scores_equals_decode_on_exact_scores(mode):
    B, H, Hkv, d = 2, 8, 2, 64
    inp = si.make_decode_inputs(B, H, Hkv, d, [300, 77], dtype="bf16", seed=21)
    q, K, V = si.as_bits(inp.q), si.as_bits(inp.K), si.as_bits(inp.V)
    sl = inp.seqlens.numpy()
    out_d, idx_d = o.santa_decode(q, K, V, sl, 40, mode, 5, 3, head_offset=8, batch_offset=1)
    qf, Kf = o.to_f64(q), o.to_f64(K)
    s = np.zeros((B, H, K.shape[2]))
    for b in range(B):
        for h in range(H):
            s[b, h, :sl[b]] = o.scores(qf[b, h], Kf[b, h // (H // Hkv), :sl[b]], 1.0 / math.sqrt(d))
    out_s, idx_s = o.santa_from_scores(s, V, sl, 40, mode, 5, 3, batch_offset=1, head_offset=8)
    np.testing.assert_array_equal(idx_s, idx_d)
    np.testing.assert_array_equal(out_s, out_d)


def test_from_scores_one_hot_is_exact_and_ignores_padding():
    B, H, Hkv, d, n = 1, 4, 2, 16, 50
    inp = si.make_decode_inputs(B, H, Hkv, d, n, dtype="bf16", seed=4)
    V = si.as_bits(inp.V)
    s = np.random.default_rng(0).normal(size=(B, H, n + 10))
    hot = [3, 49, 0, 17]
    for h, j in enumerate(hot):
        s[0, h, j] += 1e4                          # one-hot attention (logit margin 1e4)
    s[0, :, n:] = 1e6                              # positions >= seqlen must be ignored
    for mode in o.MODES:
        out, idx, det = o.santa_from_scores(s, V, [n], 64, mode, 9, return_details=True)
        for h, j in enumerate(hot):
            assert np.all(idx[0, h] == j)
            np.testing.assert_array_equal(out[0, h], o.to_f64(V[0, h // 2, j]))
            assert det["F"][(0, h)].shape == (n,)


# ---------------------------------------------------------------------------------------------
# bernoulli_scores, per-head branch (Eq. 5, tag 2)
# ---------------------------------------------------------------------------------------------

@pytest.mark.parametrize("stratified", [True, False])
def test_bernoulli_scores_per_head_branch(stratified):
    Bb, H, Hkv, d, nB = 2, 4, 2, 16, 4
    inp = si.make_decode_inputs(Bb, H, Hkv, d, [9, 4], seed=2, feature_major=True)
    sl = [9, 4]
    sc, mask = o.bernoulli_scores(si.as_bits(inp.q), si.as_bits(inp.Kt), sl, nB, stratified, False, seed=5,
                                  offset=7, batch_offset=3, head_offset=12)
    assert sc.shape == (Bb, H, 9) and mask.shape == (Bb, H, d)
    q = o.to_f64(si.as_bits(inp.q))
    Kt = o.to_f64(si.as_bits(inp.Kt))
    G = H // Hkv
    for b in range(Bb):
        assert np.all(sc[b, :, sl[b]:] == 0)
        for h in range(H):
            # the stream: Philox tag 2 (TAG_BERNOULLI_HEAD), id = global query head, global batch;
            # draws i (stratified) or i*B + n (standard), reading #1
            n_draws = d if stratified else d * nB
            u = o.philox_uniforms(5, 7, 2, 12 + h, 3 + b, np.arange(n_draws))
            if not stratified:
                u = u.reshape(d, nB)
            ph, c = o.bernoulli_qk_head(q[b, h], Kt[b, h // G, :, :sl[b]], nB, stratified, u)
            np.testing.assert_array_equal(sc[b, h, :sl[b]], ph / 4.0)   # scale = 1/sqrt(16)
            np.testing.assert_array_equal(mask[b, h], c > 0)
    # the per-head stream differs from the mean-group one (tag 3, keyed by the kv head)
    sc_g, _ = o.bernoulli_scores(si.as_bits(inp.q), si.as_bits(inp.Kt), sl, nB, stratified, True, seed=5, offset=7,
                                 batch_offset=3, head_offset=12)
    assert not np.array_equal(sc, sc_g)


def test_bernoulli_scores_per_head_exact_when_magnitudes_equal():
    """with |q_i| = norm for every i, a_i = 1, every count is B and the ternary estimator is
    exact: p_hat = q . K for every head (both draw schemes)."""
    Bb, H, Hkv, d, n = 1, 4, 2, 16, 12
    inp = si.make_decode_inputs(Bb, H, Hkv, d, n, seed=6, feature_major=True)
    rng = np.random.default_rng(1)
    qv = np.where(rng.random((Bb, H, d)) < 0.5, -0.75, 0.75).astype(np.float32)
    qb = (qv.view(np.uint32) >> 16).astype(np.uint16)           # exact in bf16
    Kt = o.to_f64(si.as_bits(inp.Kt))
    for stratified in (True, False):
        sc, mask = o.bernoulli_scores(qb, si.as_bits(inp.Kt), [n], 8, stratified, False, seed=3)
        assert mask.all()
        for h in range(H):
            exact = 0.25 * (qv[0, h].astype(np.float64) @ Kt[0, h // 2, :, :n])
            np.testing.assert_allclose(sc[0, h], exact, rtol=0, atol=1e-12)


def test_value_moments_by_second_moment_identity():
    """Sigma = E[V_J V_J^T] - mu mu^T for J ~ p, checked with exact rationals on a
    3-atom example, and tr(Sigma) = S * var_trace_iid (the iid closed form)."""
    from fractions import Fraction as Fr
    p = [Fr(1, 2), Fr(1, 3), Fr(1, 6)]
    V = [[1, 2], [-3, 0], [4, -1]]
    mu = [sum(p[j] * V[j][k] for j in range(3)) for k in range(2)]
    E2 = [[sum(p[j] * V[j][a] * V[j][b] for j in range(3)) for b in range(2)] for a in range(2)]
    Sig = [[E2[a][b] - mu[a] * mu[b] for b in range(2)] for a in range(2)]
    mu_o, Sig_o = o.value_moments(np.array([float(x) for x in p]), np.array(V, dtype=np.float64))
    np.testing.assert_allclose(mu_o, [float(x) for x in mu], rtol=0, atol=1e-14)
    np.testing.assert_allclose(Sig_o, [[float(x) for x in r] for r in Sig], rtol=0, atol=1e-13)
    assert abs(np.trace(Sig_o) - 5 * o.var_trace_iid(np.array([float(x) for x in p]), np.array(V, float), 5)) < 1e-12


def test_every_oracle_function_is_pinned_somewhere():
    """Audit behind the oracle header's claim: every public oracle function is called by name from
    at least one CPU pin file (tests/test_oracle_*.py)."""
    import glob
    import os
    import re
    root = os.path.dirname(os.path.abspath(__file__))
    src = open(os.path.join(root, "..", "oracle", "santa_oracle.py")).read()
    names = re.findall(r"^def ([a-z][a-z_0-9]*)\(", src, flags=re.M)
    pins = "".join(open(f).read() for f in glob.glob(os.path.join(root, "test_oracle_*.py")))
    missing = [n for n in names if not re.search(r"\bo\." + n + r"\b", pins)]
    assert not missing, missing
