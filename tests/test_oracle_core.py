"""Pins for the oracle's RNG, score stage, softmax, CDF, inverse CDF and gather
(-m "not gpu").  Each test checks the oracle against something other than itself."""
import math

import numpy as np
import pytest
import torch

from conftest import golden
from oracle import santa_oracle as o


def _kat_rows():
    rows = []
    for line in open(golden("philox4x32_10_kat.txt")):
        line = line.split("#")[0].strip()
        if line:
            w = [int(x, 16) for x in line.split()]
            rows.append((w[0:4], w[4:6], w[6:10]))
    return rows


def test_philox_known_answer_vectors():
    """Random123 KAT vectors (tests/golden/philox4x32_10_kat.txt)."""
    rows = _kat_rows()
    assert len(rows) == 3
    for ctr, key, want in rows:
        got = o.philox4x32_10(np.array([ctr], dtype=np.uint64), np.array(key, dtype=np.uint64))
        assert [int(x) for x in got[0]] == want


def test_philox_uniform_mapping_and_stream_layout():
    # u = r * 2^-32 exactly: draw m of the stream is word (m & 3) of block (m >> 2)
    seed, off, tag, h, b = 0x1234_5678_9ABC_DEF0, 77, 1, 5, 3
    u = o.philox_uniforms(seed, off, tag, h, b, np.arange(8))
    ctr = np.array([[0, (tag << 24) | h, b, off], [1, (tag << 24) | h, b, off]], dtype=np.uint64)
    key = np.array([seed & 0xFFFFFFFF, seed >> 32], dtype=np.uint64)
    words = o.philox4x32_10(ctr, key).reshape(-1)
    np.testing.assert_array_equal(u, words.astype(np.float64) / 2.0 ** 32)
    assert np.all(u >= 0) and np.all(u < 1)
    # different heads / batches / offsets / tags give different streams
    base = o.philox_uniforms(1, 0, 1, 0, 0, np.arange(16))
    for args in [(1, 0, 1, 1, 0), (1, 0, 1, 0, 1), (1, 1, 1, 0, 0), (1, 0, 2, 0, 0), (2, 0, 1, 0, 0)]:
        assert not np.array_equal(base, o.philox_uniforms(*args, np.arange(16)))


def test_uniform_law_of_large_numbers():
    u = o.philox_uniforms(99, 0, 1, 0, 0, np.arange(10 ** 6))
    assert 0.497 < u.mean() < 0.503
    hist = np.histogram(u, bins=16, range=(0, 1))[0]
    chi2 = ((hist - 1e6 / 16) ** 2 / (1e6 / 16)).sum()
    assert chi2 < 40.0                                              # 15 dof, p ~ 5e-4


def test_bf16_decoder_matches_torch():
    x = torch.randn(4096, dtype=torch.float32).to(torch.bfloat16)
    bits = x.view(torch.int16).numpy().view(np.uint16)
    np.testing.assert_array_equal(o.to_f64(bits), x.to(torch.float64).numpy())


def test_softmax_spec_examples():
    np.testing.assert_allclose(o.softmax([0, 0, 0, 0]), [0.25] * 4, atol=1e-15)
    np.testing.assert_allclose(o.softmax([1000, 1000]), [0.5, 0.5], atol=1e-15)
    np.testing.assert_allclose(o.softmax([math.log(1), math.log(3)]), [0.25, 0.75], atol=1e-15)
    with pytest.raises(ValueError):
        o.softmax([])
    rng = np.random.default_rng(0)
    s = rng.normal(size=50) * 1e4
    p = o.softmax(s)
    assert abs(p.sum() - 1) < 1e-12 and np.all(p >= 0)
    np.testing.assert_allclose(o.softmax(s + 123.0), p, atol=1e-12)


def test_scores_spec_examples():
    np.testing.assert_array_equal(o.scores([1, 0, 0], np.eye(3), 1.0), [1, 0, 0])
    np.testing.assert_array_equal(o.scores([1, 1], [[1, 0], [0, 1], [1, 1]], 1.0), [1, 1, 2])
    np.testing.assert_array_equal(o.scores([0, 0], [[3, 4], [5, 6]], 1.0), [0, 0])
    with pytest.raises(ValueError):
        o.scores([1, 2, 3], np.ones((4, 2)), 1.0)


def test_worked_example_eq2_3():
    """Eq. 2-3: n_k = 3, sampled one-hots (1, 1, 3) -> (V1 + V1 + V3)/3."""
    V = np.array([[1.0, 2.0, -1.0], [10.0, 20.0, 30.0], [-3.0, 0.5, 7.0]])
    got = o.gather_mean(V, np.array([0, 0, 2]))   # 0-based rows of V1, V1, V3
    np.testing.assert_allclose(got, (V[0] + V[0] + V[2]) / 3, atol=1e-15)
    # same thing written with the explicit one-hot matrix of Eq. 2
    onehots = np.array([[1, 0, 0], [1, 0, 0], [0, 0, 1]], dtype=float)
    np.testing.assert_allclose(got, (onehots.sum(0) / 3) @ V, atol=1e-15)


def test_dense_matches_torch_sdpa_fp64():
    rng = np.random.default_rng(1)
    for n, d in [(1, 8), (7, 16), (300, 64)]:
        q, K, V = rng.normal(size=d), rng.normal(size=(n, d)), rng.normal(size=(n, d))
        ref = torch.nn.functional.scaled_dot_product_attention(
            torch.tensor(q)[None, None, None], torch.tensor(K)[None, None],
            torch.tensor(V)[None, None]).numpy().reshape(-1)
        np.testing.assert_allclose(o.dense_attention(q, K, V, 1 / math.sqrt(d)), ref, atol=1e-12)


def test_dense_one_hot_and_uniform():
    rng = np.random.default_rng(2)
    V = rng.normal(size=(4, 3))
    K = np.eye(4)
    q = np.zeros(4)
    q[2] = 1e6
    np.testing.assert_array_equal(o.dense_attention(q, K, V, 1.0), V[2])
    np.testing.assert_allclose(o.dense_attention(np.zeros(4), K, V, 1.0), V.mean(0), atol=1e-15)


def test_cdf_clamp_and_inverse_cdf_convention():
    p = np.array([0.2, 0.0, 0.3, 0.5, 0.0])
    F = o.cdf(p)
    assert F[3] == 1.0 and F[4] == 1.0
    # min{j : F(j) > t}: boundary goes right; zero-mass atoms never chosen
    T = np.array([0.0, 0.1999, 0.2, 0.4999, 0.5, 0.9999999])
    np.testing.assert_array_equal(o.inverse_cdf(F, T), [0, 0, 2, 2, 3, 3])
    # brute force: exhaustive check against the defining integrand 1{F(j-1) <= t < F(j)}
    rng = np.random.default_rng(3)
    for _ in range(200):
        p = rng.dirichlet(np.ones(6)) * (rng.random(6) > 0.3)
        if p.sum() == 0:
            continue
        p /= p.sum()
        F = o.cdf(p)
        Fm1 = np.concatenate([[0.0], F[:-1]])
        for t in rng.random(20):
            j = int(o.inverse_cdf(F, [t])[0])
            hits = [i for i in range(6) if Fm1[i] <= t < F[i]]
            assert hits == [j] and p[j] > 0


def test_thresholds_definitions():
    u = np.array([0.25, 0.5, 0.75, 0.0])
    np.testing.assert_array_equal(o.thresholds("iid", 4, u), u)
    np.testing.assert_array_equal(o.thresholds("stratified", 4, u), [(0 + .25) / 4, 1.5 / 4, 2.75 / 4, 3 / 4])
    np.testing.assert_array_equal(o.thresholds("systematic", 4, u), [0.0625, 0.3125, 0.5625, 0.8125])
    with pytest.raises(ValueError):
        o.thresholds("iid", 0, u)
    # every stratified/systematic threshold lies in its stratum I_m = [m/S, (m+1)/S)
    for S in (1, 3, 7, 256):
        uu = o.philox_uniforms(5, 0, 1, 0, 0, np.arange(S))
        for mode in ("stratified", "systematic"):
            T = o.thresholds(mode, S, uu)
            m = np.arange(S)
            assert np.all(T >= m / S) and np.all(T < (m + 1) / S)


def test_unique_rows_and_fidelity():
    assert o.unique_rows(np.array([[1, 1, 3], [3, 5, 5]])) == 3
    assert o.fidelity([1, 0], [1, 0]) == (0.0, 1.0)
    r, c = o.fidelity([2, 0], [1, 0])
    assert r == 1.0 and c == 1.0
    r, c = o.fidelity([1, 0], [0, 1])
    assert abs(r - math.sqrt(2)) < 1e-15 and c == 0.0


def test_unique_rows_occupancy_formula():
    """Uniform profile, iid: E[U] = n (1 - (1 - 1/n)^S)."""
    n, S = 8192, 256
    F = o.cdf(np.full(n, 1.0 / n))
    Us = [o.unique_rows(o.inverse_cdf(F, o.philox_uniforms(s, 0, 1, 0, 0, np.arange(S))))
          for s in range(400)]
    want = n * (1 - (1 - 1 / n) ** S)
    assert abs(np.mean(Us) - want) < 0.01 * want
