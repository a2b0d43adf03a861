"""Plain fp64 CPU oracle for the SANTA / S^2ANTA decode-step hot path (arXiv 2605.01910).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this module.
The product path (``paper_2605_01910_b200``) never imports it, and it imports
nothing from the product path: the two share no code.

Everything here is slow and literal: fp64 throughout, numpy library primitives
(matmul, cumsum, searchsorted) used only as single steps of the definitions,
no blocking, no fusion, no reordering beyond what the paper states.
Citations: ``P:n`` = line n of the paper text; ``S:n`` = line n of
SPEC.md; "reading #k" = the k-th interpretation listed in DESIGN.md sec. 2.

Parity status: every public function below is pinned by a ``-m "not gpu"``
test in tests/test_oracle_*.py against something other than itself (Random123
known-answer vectors, the paper's worked example, closed forms, brute force,
exact-law enumeration, the paper's printed Bernoulli error figures).  The
validity machinery every GPU verdict rests on -- ``index_mismatch_report``
(the 1e-6 exemption rule), ``santa_from_scores`` and the per-head branch of
``bernoulli_scores`` -- is pinned in tests/test_oracle_validity.py on hand-built
cases with hand-derived verdicts.  No function here is "parity unpinned"
(audit: every ``def`` is called by name from a tests/test_oracle_*.py file).
"""
from __future__ import annotations

import math
from typing import Optional, Sequence

import numpy as np

# ---------------------------------------------------------------------------
# 0. Number formats (the oracle's own decoders; independent of any GPU code)
# ---------------------------------------------------------------------------


def to_f64(x: np.ndarray) -> np.ndarray:
    """Decode an input array to fp64.  ``uint16`` arrays are bf16 bit patterns:
    a bf16 value is the upper half of an IEEE binary32 word, so the value is the
    float32 whose bits are ``bits << 16`` (exact), then widened to fp64 (exact)."""
    x = np.asarray(x)
    if x.dtype == np.uint16:
        return (x.astype(np.uint32) << np.uint32(16)).view(np.float32).astype(np.float64)
    return x.astype(np.float64)


# ---------------------------------------------------------------------------
# 1. Counter-based RNG: Philox4x32-10 (reading #1; Salmon et al., SC'11)
# ---------------------------------------------------------------------------

PHILOX_M0 = 0xD2511F53
PHILOX_M1 = 0xCD9E8D57
PHILOX_W0 = 0x9E3779B9
PHILOX_W1 = 0xBB67AE85
_MASK32 = np.uint64(0xFFFFFFFF)

TAG_VALUE_SAMPLER = 1      # reading #1: tag 1 -> value-stage sampler thresholds
TAG_BERNOULLI_HEAD = 2     # tag 2 -> per-head Bernoulli qK^T draws
TAG_BERNOULLI_GROUP = 3    # tag 3 -> mean-group Bernoulli qK^T draws


def philox4x32_10(ctr: np.ndarray, key: np.ndarray) -> np.ndarray:
    """Philox4x32 with 10 rounds.  ``ctr``: [N, 4] uint32, ``key``: [N, 2] or [2] uint32.
    Round: (hi0,lo0)=M0*x0, (hi1,lo1)=M1*x2; x <- (hi1^x1^k0, lo1, hi0^x3^k1, lo0);
    the key is bumped by (W0, W1) between rounds."""
    c = np.asarray(ctr, dtype=np.uint64).reshape(-1, 4).copy()
    k = np.broadcast_to(np.asarray(key, dtype=np.uint64).reshape(-1, 2), (c.shape[0], 2)).copy()
    for r in range(10):
        if r > 0:
            k[:, 0] = (k[:, 0] + np.uint64(PHILOX_W0)) & _MASK32
            k[:, 1] = (k[:, 1] + np.uint64(PHILOX_W1)) & _MASK32
        p0 = np.uint64(PHILOX_M0) * c[:, 0]
        p1 = np.uint64(PHILOX_M1) * c[:, 2]
        hi0, lo0 = p0 >> np.uint64(32), p0 & _MASK32
        hi1, lo1 = p1 >> np.uint64(32), p1 & _MASK32
        c = np.stack([hi1 ^ c[:, 1] ^ k[:, 0], lo1, hi0 ^ c[:, 3] ^ k[:, 1], lo0], axis=1)
    return c.astype(np.uint32)


def philox_uniforms(seed: int, offset: int, tag: int, h_global: int, b_global: int,
                    draws: np.ndarray) -> np.ndarray:
    """Uniforms u = r * 2^-32 in [0, 1 - 2^-32] (exact in fp64) for draw indices ``draws``.
    Stream layout (reading #1): key = (seed_lo32, seed_hi32);
    counter = (draw >> 2, (tag << 24) | h_global, b_global, offset_lo32); word = draw & 3."""
    draws = np.asarray(draws, dtype=np.uint64).reshape(-1)
    n = draws.shape[0]
    ctr = np.zeros((n, 4), dtype=np.uint64)
    ctr[:, 0] = draws >> np.uint64(2)
    ctr[:, 1] = (np.uint64(tag) << np.uint64(24)) | np.uint64(h_global & 0xFFFFFF)
    ctr[:, 2] = np.uint64(b_global & 0xFFFFFFFF)
    ctr[:, 3] = np.uint64(offset & 0xFFFFFFFF)
    key = np.array([seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF], dtype=np.uint64)
    out = philox4x32_10(ctr, key)
    words = out[np.arange(n), (draws & np.uint64(3)).astype(np.int64)]
    return words.astype(np.float64) * 2.0 ** -32


# ---------------------------------------------------------------------------
# 2. Score stage, softmax, CDF (Eq. 1)
# ---------------------------------------------------------------------------


def scores(q: np.ndarray, K: np.ndarray, scale: float) -> np.ndarray:
    """s_n = (q . K_n) * scale for every key row n (Eq. 1).
    q: [d], K: [n, d] (fp64)."""
    q = np.asarray(q, dtype=np.float64)
    K = np.asarray(K, dtype=np.float64)
    if q.shape[-1] != K.shape[-1]:
        raise ValueError("dimension mismatch")
    return (K @ q) * scale


def softmax(s: np.ndarray) -> np.ndarray:
    """Numerically stable softmax, p_n = exp(s_n - max s) / sum_m exp(s_m - max s)."""
    s = np.asarray(s, dtype=np.float64)
    if s.size == 0:
        raise ValueError("empty distribution")
    e = np.exp(s - s.max())
    return e / e.sum()


def cdf(p: np.ndarray) -> np.ndarray:
    """F(j) = sum_{i<=j} p_i, accumulated sequentially in fp64, then clamped to exactly 1
    from the last index with positive mass onward (reading #5)."""
    F = np.cumsum(np.asarray(p, dtype=np.float64))
    pos = np.nonzero(np.asarray(p) > 0)[0]
    if pos.size:
        F[pos[-1]:] = 1.0
    return F


def inverse_cdf(F: np.ndarray, T: np.ndarray) -> np.ndarray:
    """J = F^{-1}(T) = min{ j : F(j) > T } (reading #4: the integrand convention
    1{F(j-1) <= t < F(j)} of P:699).  A threshold on a boundary goes right;
    zero-mass atoms are never selected."""
    return np.searchsorted(F, np.asarray(T, dtype=np.float64), side="right").astype(np.int64)


# ---------------------------------------------------------------------------
# 3. Thresholds of the three samplers
# ---------------------------------------------------------------------------

MODES = ("iid", "stratified", "systematic")


def thresholds(mode: str, S: int, u: np.ndarray) -> np.ndarray:
    """Thresholds T_m, m = 0..S-1, from uniforms u (fp64, exact):
    * iid        (SANTA):            T_m = u_m                (S fresh uniforms)
    * stratified (S^2ANTA-strat):   T_m = (m + u_m) / S      (T_m ~ Unif(I_m), I_m=[m/S,(m+1)/S))
    * systematic (S^2ANTA-sys):     T_m = (m + u_0) / S      (one U = u_0/S ~ Unif[0,1/S); reading #2)
    """
    if S < 1:
        raise ValueError("empty budget")
    m = np.arange(S, dtype=np.float64)
    u = np.asarray(u, dtype=np.float64)
    if mode == "iid":
        return u[:S].copy()
    if mode == "stratified":
        return (m + u[:S]) / S
    if mode == "systematic":
        return (m + u[0]) / S
    raise ValueError(f"unknown mode {mode}")


def sampler_uniforms(mode: str, S: int, seed: int, offset: int, h_global: int,
                     b_global: int) -> np.ndarray:
    """The uniforms each sampler consumes from the value-sampler Philox stream (tag 1):
    draws 0..S-1 for iid/stratified, draw 0 only for systematic (one random number per
    query)."""
    n = 1 if mode == "systematic" else S
    return philox_uniforms(seed, offset, TAG_VALUE_SAMPLER, h_global, b_global, np.arange(n))


def systematic_counts_formula(F: np.ndarray, S: int, u: float) -> np.ndarray:
    """Second, independent route to systematic sampling: the per-key count form of
    Pass-2 (Alg. prop-pass2): c_n = floor(a0 + S F(n)) - floor(a0 + S F(n-1)),
    applied to the GLOBAL CDF with a0 = 1 - u (reading #9; equal to the search route
    except on exact ties)."""
    a0 = 1.0 - u
    SF = S * np.concatenate([[0.0], np.asarray(F, dtype=np.float64)])
    return (np.floor(a0 + SF[1:]) - np.floor(a0 + SF[:-1])).astype(np.int64)


# ---------------------------------------------------------------------------
# 4. Value stage (Eq. 4; worked example Eqs. 2-3)
# ---------------------------------------------------------------------------


def gather_mean(V: np.ndarray, idx: np.ndarray) -> np.ndarray:
    """out = (1/S) sum_s V_{i_s} (Eq. 4), fp64 adds then one multiply by 1/S
    (reading #7; the bit-shift remark P:112 is not emulated)."""
    V = np.asarray(V, dtype=np.float64)
    idx = np.asarray(idx, dtype=np.int64)
    S = idx.shape[0]
    if S < 1:
        raise ValueError("empty budget")
    acc = np.zeros(V.shape[1], dtype=np.float64)
    for i in idx:
        acc += V[i]
    return acc * (1.0 / S)


def dense_attention(q, K, V, scale) -> np.ndarray:
    """Exact SDPA decode output softmax(q K^T * scale) V (Eq. 1)."""
    p = softmax(scores(q, K, scale))
    return p @ np.asarray(V, dtype=np.float64)


def santa_estimate(q, K, V, scale, S, mode, u) -> tuple[np.ndarray, np.ndarray]:
    """One query's SANTA / S^2ANTA estimate: scores -> softmax -> CDF ->
    thresholds from uniforms ``u`` -> inverse CDF -> (1/S) sum of V rows.
    Returns (out [d], idx [S])."""
    p = softmax(scores(q, K, scale))
    F = cdf(p)
    T = thresholds(mode, S, u)
    idx = inverse_cdf(F, T)
    return gather_mean(V, idx), idx


# ---------------------------------------------------------------------------
# 5. Batched decode step over (b, h) with GQA (k(h) = floor(h/G))
# ---------------------------------------------------------------------------


def _seq_kv(Kl: np.ndarray, b: int, kv: int, n: int) -> np.ndarray:
    return to_f64(Kl[b, kv, :n, :])


def santa_decode(q, K, V, seqlens, S: int, mode: str, seed: int, offset: int = 0,
                 scale: Optional[float] = None, batch_offset: int = 0, head_offset: int = 0,
                 return_details: bool = False):
    """The whole decode step the C-ABI ``santa_decode_attention`` computes, for every
    batch b and query head h: kv = floor(h/G), n = seqlens[b] (reading #10: seqlens
    include the current token), s = (q_h . K_{kv,j}) * scale for j < n, p = softmax(s),
    F = CDF, T = thresholds(Philox stream of global (b, h)), J = F^{-1}(T),
    out = (1/S) sum_m V_{kv, J_m}.

    q: [B, H, d]; K, V: [B, H_kv, n_max, d] logical layout (bf16 as uint16 bits, or float).
    Returns out [B, H, d] fp64 and idx [B, H, S] int64 (and details if requested)."""
    qf = to_f64(q)
    B, H, d = qf.shape
    Hkv = K.shape[1]
    G = H // Hkv
    scale = 1.0 / math.sqrt(d) if not scale else scale
    out = np.zeros((B, H, d))
    idx = np.zeros((B, H, S), dtype=np.int64)
    det = {"F": {}, "T": {}}
    for b in range(B):
        n = int(seqlens[b])
        if n < 1:
            raise ValueError("empty distribution")
        for h in range(H):
            kv = h // G
            Kb = _seq_kv(K, b, kv, n)
            Vb = _seq_kv(V, b, kv, n)
            u = sampler_uniforms(mode, S, seed, offset, head_offset + h, batch_offset + b)
            p = softmax(scores(qf[b, h], Kb, scale))
            F = cdf(p)
            T = thresholds(mode, S, u)
            J = inverse_cdf(F, T)
            out[b, h] = gather_mean(Vb, J)
            idx[b, h] = J
            if return_details:
                det["F"][(b, h)] = F
                det["T"][(b, h)] = T
    if return_details:
        return out, idx, det
    return out, idx


def dense_decode(q, K, V, seqlens, scale: Optional[float] = None) -> np.ndarray:
    """Exact dense decode for every (b, h): softmax(q K^T scale) V over j < seqlens[b]."""
    qf = to_f64(q)
    B, H, d = qf.shape
    G = H // K.shape[1]
    scale = 1.0 / math.sqrt(d) if not scale else scale
    out = np.zeros((B, H, d))
    for b in range(B):
        n = int(seqlens[b])
        for h in range(H):
            kv = h // G
            out[b, h] = dense_attention(qf[b, h], _seq_kv(K, b, kv, n), _seq_kv(V, b, kv, n), scale)
    return out


def out_given_idx(V, idx) -> np.ndarray:
    """(1/S) sum_m V_{kv(h), idx[b,h,m]} in fp64 for GIVEN indices -- used to compare the
    GPU's output on the GPU's own indices (reading #16)."""
    B, H, S = idx.shape
    G = H // V.shape[1]
    out = np.zeros((B, H, V.shape[3]))
    for b in range(B):
        for h in range(H):
            out[b, h] = gather_mean(to_f64(V[b, h // G]), idx[b, h])
    return out


def index_mismatch_report(F_by_bh: dict, T_by_bh: dict, idx_oracle, idx_gpu, tol: float = 1e-6):
    """Reading #19: a sample whose oracle index j_o differs from the GPU index j_g is
    EXEMPT iff every oracle CDF boundary F(j), j in [min, max), lies within ``tol`` of
    its threshold T.  Returns (n_total, n_mismatch, n_exempt, list_of_failures)."""
    idx_oracle = np.asarray(idx_oracle)
    idx_gpu = np.asarray(idx_gpu)
    B, H, S = idx_oracle.shape
    mism = exempt = 0
    fails = []
    for b in range(B):
        for h in range(H):
            F = F_by_bh[(b, h)]
            T = T_by_bh[(b, h)]
            for m in np.nonzero(idx_oracle[b, h] != idx_gpu[b, h])[0]:
                mism += 1
                jo, jg = int(idx_oracle[b, h, m]), int(idx_gpu[b, h, m])
                lo, hi = min(jo, jg), max(jo, jg)
                if 0 <= lo and hi <= len(F) and np.all(np.abs(F[lo:hi] - T[m]) < tol):
                    exempt += 1
                else:
                    fails.append((b, h, int(m), jo, jg, float(T[m])))
    return B * H * S, mism, exempt, fails


# ---------------------------------------------------------------------------
# 6. Exact laws and variances
# ---------------------------------------------------------------------------


def value_moments(p, V):
    """mu = sum_j p_j V_j and Sigma = sum_j p_j (V_j - mu)(V_j - mu)^T."""
    p = np.asarray(p, dtype=np.float64)
    V = np.asarray(V, dtype=np.float64)
    mu = p @ V
    D = V - mu
    return mu, (D * p[:, None]).T @ D


def var_trace_iid(p, V, S) -> float:
    """VarTrace_multi = tr(Sigma)/S, tr(Sigma) = sum_j p_j ||V_j||^2 - ||mu||^2."""
    p = np.asarray(p, dtype=np.float64)
    V = np.asarray(V, dtype=np.float64)
    mu = p @ V
    return float((p @ (V * V).sum(1) - mu @ mu) / S)


def stratum_law(p, S) -> np.ndarray:
    """P(J_m = j) for stratified sampling: T_m ~ Unif(I_m), so
    P(J_m = j) = S * |[F(j-1), F(j)) cap [m/S, (m+1)/S)|. Shape [S, n]."""
    F = cdf(p)
    Fm1 = np.concatenate([[0.0], F[:-1]])
    lo = np.arange(S)[:, None] / S
    hi = (np.arange(S)[:, None] + 1) / S
    return S * np.clip(np.minimum(F[None, :], hi) - np.maximum(Fm1[None, :], lo), 0.0, None)


def var_stratified(p, V, S):
    """Per-coordinate variance and trace of S^2ANTA-strat: (1/S^2) sum_m Var(V_{J_m})
    with the within-stratum law above (Thm P:710-722)."""
    V = np.asarray(V, dtype=np.float64)
    W = stratum_law(p, S)
    mu_m = W @ V
    var_m = W @ (V * V) - mu_m * mu_m
    per_coord = var_m.sum(0) / S ** 2
    return per_coord, float(per_coord.sum())


def systematic_law(p, V, S):
    """Exact law of S^2ANTA-sys by a breakpoint sweep over the single uniform u in [0,1):
    T_m = (m+u)/S, so the index vector J(u) only changes where u = S F(j) - m, i.e. at
    u = frac(S F(j)).  Between consecutive breakpoints J(u) is constant, so
    E[out] and E[out^2] are exact finite sums (the replicate estimator of
    P:1380-1391 is the paper's approximation of this).  Returns (mean, per_coord_var)."""
    V = np.asarray(V, dtype=np.float64)
    F = cdf(p)
    bps = np.unique(np.concatenate([[0.0, 1.0], np.mod(S * F, 1.0)]))
    bps = bps[(bps >= 0.0) & (bps <= 1.0)]
    m = np.arange(S)
    mean = np.zeros(V.shape[1])
    sq = np.zeros(V.shape[1])
    for a, c in zip(bps[:-1], bps[1:]):
        w = c - a
        if w <= 0:
            continue
        u = 0.5 * (a + c)
        J = inverse_cdf(F, (m + u) / S)
        o = V[J].sum(0) / S
        mean += w * o
        sq += w * o * o
    return mean, sq - mean * mean


def var_iid_per_coord(p, V, S):
    """Per-coordinate variance of iid SANTA: diag(Sigma)/S."""
    mu, Sig = value_moments(p, V)
    return np.diag(Sig) / S


# ---------------------------------------------------------------------------
# 7. Bernoulli qK^T score stage (Eq. 5; App. C)
# ---------------------------------------------------------------------------


def bernoulli_counts(a: np.ndarray, B: int, stratified: bool, u: np.ndarray) -> np.ndarray:
    """Per-feature counts c_i = sum_n b_i^(n) of B Bernoulli(a_i) draws.
    * standard:  c_i = #{ n < B : u_{i,n} < a_i },  u: [d, B]
    * stratified (reading #11): c_i = floor(B a_i) + 1[u_i < B a_i - floor(B a_i)], u: [d]
    All comparisons in fp64."""
    a = np.asarray(a, dtype=np.float64)
    if B < 1:
        raise ValueError("B must be >= 1")
    if stratified:
        Ba = B * a
        fl = np.floor(Ba)
        return (fl + (np.asarray(u).reshape(-1) < (Ba - fl))).astype(np.int64)
    return (np.asarray(u).reshape(a.shape[0], B) < a[:, None]).sum(1).astype(np.int64)


def _bern_uniforms(B, stratified, d, seed, offset, tag, id_global, b_global):
    if stratified:
        return philox_uniforms(seed, offset, tag, id_global, b_global, np.arange(d))
    return philox_uniforms(seed, offset, tag, id_global, b_global, np.arange(d * B)).reshape(d, B)


def bernoulli_qk_head(q, Kt, B, stratified, u):
    """Per-head ternary estimator (Eq. 5; App. C):
    norm = max_i |q_i| (reading #12), a_i = |q_i|/norm, q_hat^(n)_i = b_i^(n) sign(q_i),
    p_hat = (norm/B) sum_n q_hat^(n) K^T = (norm/B) sum_i c_i sign(q_i) K^T_i.
    q: [d] fp64, Kt: [d, n] fp64 feature-major.  Returns (p_hat [n], counts [d])."""
    q = np.asarray(q, dtype=np.float64)
    norm = np.abs(q).max()
    if norm == 0.0:
        return np.zeros(Kt.shape[1]), np.zeros(q.shape[0], dtype=np.int64)
    c = bernoulli_counts(np.abs(q) / norm, B, stratified, u)
    w = (norm / B) * c * np.sign(q)
    sel = np.nonzero(c)[0]
    return w[sel] @ np.asarray(Kt, dtype=np.float64)[sel], c


def bernoulli_qk_mean_group(qg, Kt, B, stratified, u):
    """Mean-group-query estimator (Eq. 6; App. C.2):
    m_i = (1/G) sum_g |q_{g,i}|, norm = max_i m_i (reading #12), b_i ~ Bernoulli(m_i/norm),
    m_hat = (norm/B) sum_n b^(n) = norm c / B, p_hat_g = (m_hat . q_g / m) K^T over the
    selected features {i : c_i > 0, m_i > 0} (reading #14).
    qg: [G, d], Kt: [d, n].  Returns (p_hat [G, n], counts [d])."""
    qg = np.asarray(qg, dtype=np.float64)
    G, d = qg.shape
    m = np.abs(qg).sum(0) / G
    norm = m.max()
    if norm == 0.0:
        return np.zeros((G, Kt.shape[1])), np.zeros(d, dtype=np.int64)
    c = bernoulli_counts(m / norm, B, stratified, u)
    sel = np.nonzero((c > 0) & (m > 0))[0]
    mhat = norm * c[sel] / B
    w = mhat[None, :] * qg[:, sel] / m[None, sel]
    return w @ np.asarray(Kt, dtype=np.float64)[sel], c


def bernoulli_scores(q, Kt, seqlens, B: int, stratified: bool, mean_group: bool, seed: int,
                     offset: int = 0, scale: Optional[float] = None, batch_offset: int = 0,
                     head_offset: int = 0):
    """What ``santa_bernoulli_scores`` computes: scale * p_hat for every (b, h) over
    j < seqlens[b] (positions >= seqlen are 0).  Kt: [B, H_kv, d, n_max] feature-major.
    Returns (scores [B, H, n_max] fp64, feature_mask [B, H_kv or H, d] bool)."""
    qf = to_f64(q)
    Bb, H, d = qf.shape
    Hkv = Kt.shape[1]
    G = H // Hkv
    n_max = Kt.shape[3]
    scale = 1.0 / math.sqrt(d) if not scale else scale
    out = np.zeros((Bb, H, n_max))
    mask = np.zeros((Bb, Hkv if mean_group else H, d), dtype=bool)
    for b in range(Bb):
        n = int(seqlens[b])
        for kv in range(Hkv):
            Ktb = to_f64(Kt[b, kv, :, :n])
            if mean_group:
                u = _bern_uniforms(B, stratified, d, seed, offset, TAG_BERNOULLI_GROUP,
                                   head_offset // G + kv, batch_offset + b)
                ph, c = bernoulli_qk_mean_group(qf[b, kv * G:(kv + 1) * G], Ktb, B, stratified, u)
                out[b, kv * G:(kv + 1) * G, :n] = scale * ph
                mask[b, kv] = c > 0
            else:
                for g in range(G):
                    h = kv * G + g
                    u = _bern_uniforms(B, stratified, d, seed, offset, TAG_BERNOULLI_HEAD,
                                       head_offset + h, batch_offset + b)
                    ph, c = bernoulli_qk_head(qf[b, h], Ktb, B, stratified, u)
                    out[b, h, :n] = scale * ph
                    mask[b, h] = c > 0
    return out, mask


def santa_from_scores(s_bh: np.ndarray, V, seqlens, S, mode, seed, offset=0, batch_offset=0,
                      head_offset=0, return_details=False):
    """Value stage on GIVEN scores (the config-5 combination):
    softmax over s[b, h, :n] -> CDF -> thresholds -> inverse CDF -> mean of V rows."""
    Bb, H, _ = s_bh.shape
    G = H // V.shape[1]
    out = np.zeros((Bb, H, V.shape[3]))
    idx = np.zeros((Bb, H, S), dtype=np.int64)
    det = {"F": {}, "T": {}}
    for b in range(Bb):
        n = int(seqlens[b])
        for h in range(H):
            F = cdf(softmax(s_bh[b, h, :n]))
            T = thresholds(mode, S, sampler_uniforms(mode, S, seed, offset, head_offset + h,
                                                     batch_offset + b))
            J = inverse_cdf(F, T)
            out[b, h] = gather_mean(to_f64(V[b, h // G, :n]), J)
            idx[b, h] = J
            det["F"][(b, h)] = F
            det["T"][(b, h)] = T
    if return_details:
        return out, idx, det
    return out, idx


# ---------------------------------------------------------------------------
# 8. Sequence-sharded sampling (reading #18; no paper passage -- extension)
# ---------------------------------------------------------------------------


def shard_bounds(n: int, R: int) -> list[tuple[int, int]]:
    """Contiguous shards in rank order: rank r holds tokens [r*n//R, (r+1)*n//R)."""
    return [(r * n // R, (r + 1) * n // R) for r in range(R)]


def shard_stats(s: np.ndarray) -> tuple[float, float]:
    """Local softmax statistics of one shard's scores: (m_r, Lambda_r = sum exp(s - m_r));
    an empty shard gives (-inf, 0)."""
    if s.size == 0:
        return -math.inf, 0.0
    m = float(s.max())
    return m, float(np.exp(s - m).sum())


def shard_sample(s_local: np.ndarray, token_offset: int, stats_all, rank: int,
                 T: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """Rank ``rank`` keeps the thresholds that fall in its slice of the global CDF:
    W_r = exp(m_r - m*) Lambda_r, Z = sum_r W_r, F_r = sum_{r'<=r} W_r'/Z; sample m is
    local iff F_{r-1} <= T_m < F_r; its index is the local inverse CDF of
    (T_m - F_{r-1}) Z / W_r on the local softmax.  Returns (strata m, global token ids)."""
    ms = np.array([st[0] for st in stats_all])
    Ls = np.array([st[1] for st in stats_all])
    mstar = ms.max()
    W = np.where(Ls > 0, np.exp(ms - mstar) * Ls, 0.0)
    Z = W.sum()
    Fr = np.cumsum(W) / Z
    pos = np.nonzero(W > 0)[0]
    Fr[pos[-1]:] = 1.0
    lo = 0.0 if rank == 0 else Fr[rank - 1]
    hi = Fr[rank]
    mine = np.nonzero((T >= lo) & (T < hi))[0]
    if mine.size == 0 or W[rank] == 0:
        return mine, np.zeros(0, dtype=np.int64)
    tloc = (T[mine] - lo) * Z / W[rank]
    Floc = cdf(softmax(s_local))
    return mine, token_offset + inverse_cdf(Floc, tloc)


# ---------------------------------------------------------------------------
# 9. Measurement instruments (App. N)
# ---------------------------------------------------------------------------


def unique_rows(idx_group: np.ndarray) -> int:
    """U = |{J}| over all samples of a GQA group (union over heads)."""
    return int(np.unique(np.asarray(idx_group).reshape(-1)).size)


def fidelity(approx, exact) -> tuple[float, float]:
    """Relative L2 error and cosine similarity."""
    a = np.asarray(approx, dtype=np.float64).reshape(-1)
    e = np.asarray(exact, dtype=np.float64).reshape(-1)
    ne = np.linalg.norm(e)
    if ne == 0:
        raise ValueError("undefined relative error")
    return float(np.linalg.norm(a - e) / ne), float(a @ e / (np.linalg.norm(a) * ne))


# ---------------------------------------------------------------------------
# 9. S^2ANTA-prop with largest-remainder tile budgets (
#    App. M, Alg. prop-pass1, Alg. prop-budgets P:1597-1613,
#    Alg. prop-pass2; mini version P:1556-1573)
# ---------------------------------------------------------------------------

TAG_PROP_TILE_OFFSET = 4   # reading #25: tag 4 -> a_{0,h,t}, draw index = tile t


def prop_tile_stats(s: np.ndarray, B_tile: int):
    """Kernel 1: T = ceil(n_k / B_tile) tiles T_t = [t B_tile, min((t+1) B_tile, n_k));
    m_t = max_{n in T_t} s_n, l_t = sum_{n in T_t} exp(s_n - m_t), u_n = exp(s_n - m_t) (the optional
    u-stash).  Returns (m [T], l [T], u [n_k]) in fp64."""
    s = np.asarray(s, dtype=np.float64)
    n = s.shape[0]
    if n < 1 or B_tile < 1:
        raise ValueError("empty distribution")
    T = -(-n // B_tile)
    m = np.empty(T)
    l = np.empty(T)
    u = np.empty(n)
    for t in range(T):
        lo, hi = t * B_tile, min((t + 1) * B_tile, n)
        m[t] = s[lo:hi].max()
        u[lo:hi] = np.exp(s[lo:hi] - m[t])
        l[t] = u[lo:hi].sum()
    return m, l, u


def largest_remainder(q: np.ndarray, S: int) -> np.ndarray:
    """S_t = floor(q_t), then the remaining S - sum_t S_t samples one each to the tiles with the
    largest fractional part of q_t; equal fractional parts go to the lower tile
    index (reading #25).  q: quotas [T] fp64 summing to S."""
    q = np.asarray(q, dtype=np.float64)
    fl = np.floor(q)
    St = fl.astype(np.int64)
    R = S - int(St.sum())
    if R < 0 or R > q.shape[0]:
        raise ValueError("quotas do not sum to S")
    frac = q - fl
    order = sorted(range(q.shape[0]), key=lambda t: (-frac[t], t))
    for t in order[:R]:
        St[t] += 1
    return St


def prop_budgets(m: np.ndarray, l: np.ndarray, S: int):
    """Kernel 2 for one head: m* = max_t m_t, W_t = exp(m_t - m*) l_t, Z = sum_t W_t,
    q_t = S W_t / Z, S_t = largest_remainder(q, S), invdelta_t = S_t / l_t if S_t > 0 else 0.
    Returns (S_t [T] int64, invdelta [T], q [T])."""
    m = np.asarray(m, dtype=np.float64)
    l = np.asarray(l, dtype=np.float64)
    mstar = m.max()
    W = np.exp(m - mstar) * l
    Z = W.sum()
    q = S * W / Z
    St = largest_remainder(q, S)
    invd = np.where(St > 0, St / np.where(l > 0, l, 1.0), 0.0)
    return St, invd, q


def prop_counts(u: np.ndarray, B_tile: int, invdelta: np.ndarray, a0: np.ndarray) -> np.ndarray:
    """Kernel 3 counts, literally: per tile, p = 0; for n increasing:
    x = invdelta_t u_n; c_n = floor(a0_t + p + x) - floor(a0_t + p); p += x."""
    n = u.shape[0]
    c = np.zeros(n, dtype=np.int64)
    for t in range(invdelta.shape[0]):
        p = 0.0
        for i in range(t * B_tile, min((t + 1) * B_tile, n)):
            x = invdelta[t] * u[i]
            c[i] = int(math.floor(a0[t] + p + x) - math.floor(a0[t] + p))
            p += x
    return c


def santa_prop_decode(q, K, V, seqlens, S: int, seed: int, offset: int = 0, B_tile: int = 64,
                      scale: Optional[float] = None, batch_offset: int = 0, head_offset: int = 0,
                      return_details: bool = False):
    """The S^2ANTA-prop decode step (Alg. prop-mini) for every (b, h), kv = floor(h/G):
    scores over j < seqlens[b] -> Kernel 1 tile stats -> Kernel 2 budgets (a0_t = Philox tag 4,
    draw t, reading #25) -> Kernel 3 counts -> O = sum_n c_n V_n, out = O / S.
    idx [B, H, S]: the emitted rows, tile-major, each row repeated c_n times (the GPU's order).
    Returns out [B, H, d] fp64, idx (and details {(b,h): (St, q, a0, c)} if requested)."""
    qf = to_f64(q)
    B, H, d = qf.shape
    G = H // K.shape[1]
    scale = 1.0 / math.sqrt(d) if not scale else scale
    out = np.zeros((B, H, d))
    idx = np.zeros((B, H, S), dtype=np.int64)
    det = {}
    for b in range(B):
        n = int(seqlens[b])
        if n < 1:
            raise ValueError("empty distribution")
        for h in range(H):
            kv = h // G
            Kb = _seq_kv(K, b, kv, n)
            Vb = _seq_kv(V, b, kv, n)
            s = scores(qf[b, h], Kb, scale)
            m, l, u = prop_tile_stats(s, B_tile)
            St, invd, qt = prop_budgets(m, l, S)
            a0 = philox_uniforms(seed, offset, TAG_PROP_TILE_OFFSET, head_offset + h, batch_offset + b,
                                 np.arange(m.shape[0]))
            c = prop_counts(u, B_tile, invd, a0)
            J = np.repeat(np.arange(n), c)
            if J.shape[0] != S:
                raise ValueError("emitted sample count differs from S")
            acc = np.zeros(d)
            for i in np.nonzero(c)[0]:
                acc += c[i] * Vb[i]
            out[b, h] = acc / S
            idx[b, h] = J
            if return_details:
                det[(b, h)] = {"St": St, "q": qt, "a0": a0, "c": c, "m": m, "l": l, "u": u}
    if return_details:
        return out, idx, det
    return out, idx


# ---------------------------------------------------------------------------
# 10. S^2ANTA-flash: uniform per-tile budgets + deferred LSE merge (
#     App. N: overview P:1651-1667, Kernel 1 P:1669-1689, Kernel 2 P:1691-1706)
# ---------------------------------------------------------------------------

TAG_FLASH_TILE_OFFSET = 5  # reading #26: tag 5 -> flash a_{0,h,t}, draw index = tile t


def flash_tile_budget(n: int, B_tile: int, S: int) -> int:
    """S_tile ~ S / T 'rounded', T = ceil(n_k / B_tile): round half up, at least 1
    (reading #26 -- a tile with budget 0 would drop its mass from the estimator)."""
    T = -(-n // B_tile)
    return max(1, int(math.floor(S / T + 0.5)))


def flash_merge(m: np.ndarray, l: np.ndarray, O_tilde: np.ndarray, S_tile: int) -> np.ndarray:
    """Kernel 2: m* = max_t m_t, W_t = exp(m_t - m*) l_t, Z = sum_t W_t,
    O = (1/Z) sum_t W_t (O~_t / S_tile)."""
    m = np.asarray(m, dtype=np.float64)
    l = np.asarray(l, dtype=np.float64)
    W = np.exp(m - m.max()) * l
    Z = W.sum()
    return (W[:, None] * (np.asarray(O_tilde, dtype=np.float64) / S_tile)).sum(0) / Z


def santa_flash_decode(q, K, V, seqlens, S: int, seed: int, offset: int = 0, B_tile: int = 256,
                       scale: Optional[float] = None, batch_offset: int = 0, head_offset: int = 0,
                       return_details: bool = False):
    """The S^2ANTA-flash decode step for every (b, h), kv = floor(h/G): Kernel 1 per tile
    m_t, u_n = exp(s_n - m_t), l_t, invdelta_t = S_tile / l_t, a0_t = Philox tag 5 draw t, systematic
    counts c_n (the same loop as prop-pass2), O~_t = sum_{n in T_t} c_n V_n; Kernel 2
    flash_merge.  idx [B, H, M_max]: the rows drawn (tile-major, each c_n times; M_b = S_tile(b) T_b,
    padded with -1).  Returns out [B, H, d] fp64, idx (and details if requested)."""
    qf = to_f64(q)
    B, H, d = qf.shape
    G = H // K.shape[1]
    scale = 1.0 / math.sqrt(d) if not scale else scale
    Mmax = max(flash_tile_budget(int(n), B_tile, S) * -(-int(n) // B_tile) for n in seqlens)
    out = np.zeros((B, H, d))
    idx = np.full((B, H, Mmax), -1, dtype=np.int64)
    det = {}
    for b in range(B):
        n = int(seqlens[b])
        if n < 1:
            raise ValueError("empty distribution")
        S_tile = flash_tile_budget(n, B_tile, S)
        for h in range(H):
            kv = h // G
            Kb = _seq_kv(K, b, kv, n)
            Vb = _seq_kv(V, b, kv, n)
            s = scores(qf[b, h], Kb, scale)
            m, l, u = prop_tile_stats(s, B_tile)
            T = m.shape[0]
            invd = S_tile / l
            a0 = philox_uniforms(seed, offset, TAG_FLASH_TILE_OFFSET, head_offset + h, batch_offset + b,
                                 np.arange(T))
            c = prop_counts(u, B_tile, invd, a0)
            O_t = np.zeros((T, d))
            for i in np.nonzero(c)[0]:
                O_t[i // B_tile] += c[i] * Vb[i]
            out[b, h] = flash_merge(m, l, O_t, S_tile)
            J = np.repeat(np.arange(n), c)
            idx[b, h, :J.shape[0]] = J
            if return_details:
                det[(b, h)] = {"S_tile": S_tile, "a0": a0, "c": c, "m": m, "l": l, "u": u}
    if return_details:
        return out, idx, det
    return out, idx
