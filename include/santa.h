/*
 * santa.h -- C ABI of libsanta.so: SANTA / S^2ANTA stochastic sparse decode-step
 * attention (arXiv 2605.01910) for NVIDIA B200 (sm_100a).
 *
 * Citations: "P:n" = line n of the paper text; "S:n" = SPEC.md line n;
 * "reading #k" = the k-th interpretation of the paper listed in DESIGN.md sec. 2.
 *
 * Conventions shared by every entry point
 * ---------------------------------------
 * - All tensor pointers are DEVICE pointers unless the name ends in _host.  The
 *   caller owns every buffer; the library never allocates or frees device memory.
 *   Its only process-wide state is a cache of per-(kernel, device) launch attributes
 *   and per-device SM counts, guarded by a mutex and written idempotently, so calls
 *   from several host threads on different streams (and devices) are reentrant.
 * - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *   Calls are stream-ordered and asynchronous: a return of SANTA_OK means the
 *   work was launched, not that it finished.
 * - Arguments are validated synchronously on the host BEFORE anything is
 *   launched.  On any error nothing is launched and no output is touched.  No
 *   exception or abort crosses the ABI.  No host<->device synchronisation happens
 *   inside any call except santa_read_error_flags, santa_decode_step_host and
 *   santa_decode_step_host_packed with synchronize != 0.
 * - Determinism: identical inputs, seed and offset give bit-identical `out` and
 *   `idx_out` across runs (no floating-point atomics anywhere).
 * - Device-side data errors (a seqlen < 1, i.e. an "empty distribution")
 *   cannot be seen on the host without a sync: the kernels write zeros to that
 *   sequence's outputs and set bit SANTA_FLAG_EMPTY_SEQ in the workspace flag
 *   word, readable with santa_read_error_flags() after the stream is synced.
 *
 * Layout of the KV cache (the paper's cache is sequence-major [n_k+1, H_kv, d],
 * P:1752; ours is head-major and optionally paged -- DESIGN.md sec. 4):
 * - contiguous (page_table == NULL): K, V are [batch, n_kv_heads, max_seqlen, head_dim]
 * - paged      (page_table != NULL): K, V are pools [num_pages, n_kv_heads, page_size, head_dim];
 *   page_table is int32 [batch, max_pages_per_seq]; logical page i of sequence b is
 *   physical page page_table[b*max_pages_per_seq + i]; token t lives in logical
 *   page t / page_size at row t % page_size.
 * - seqlens is a device int32 [batch]; seqlens[b] counts every cached token
 *   INCLUDING the current one (reading #10); keys at positions >= seqlens[b]
 *   are masked (zero mass).
 * - q, out are [batch, n_heads, head_dim]; query head h attends kv head floor(h/G),
 *   G = n_heads / n_kv_heads (GQA).
 */
#ifndef SANTA_H_
#define SANTA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

typedef enum {
  SANTA_OK = 0,
  SANTA_ERR_INVALID_ARG = 1,        /* NULL pointer, bad enum, bad scale, ...            */
  SANTA_ERR_SHAPE = 2,              /* H % H_kv != 0, non-positive sizes, page geometry   */
  SANTA_ERR_EMPTY_BUDGET = 3,       /* S < 1  (SPEC "empty budget") or B < 1 */
  SANTA_ERR_EMPTY_DISTRIBUTION = 4, /* max_seqlen < 1 (SPEC "empty distribution")   */
  SANTA_ERR_UNSUPPORTED = 5,        /* head_dim not in {64,128}, G > 8, dtype combination */
  SANTA_ERR_WORKSPACE = 6,          /* workspace NULL, too small or not 256-B aligned     */
  SANTA_ERR_ALIGNMENT = 7,          /* a tensor pointer not 16-byte aligned               */
  SANTA_ERR_CUDA = 8                /* a CUDA launch/runtime call failed                  */
} santa_status;

typedef enum {
  SANTA_IID = 0,         /* SANTA: S i.i.d. categorical draws, T_m = u_m (Eq. 4)          */
  SANTA_STRATIFIED = 1,  /* S^2ANTA-strat: T_m = (m + u_m)/S, independent u_m                */
  SANTA_SYSTEMATIC = 2   /* S^2ANTA-sys: T_m = (m + u_0)/S, one uniform per (b, h) (reading #2) */
} santa_mode;

typedef enum { SANTA_BF16 = 0, SANTA_F32 = 1, SANTA_F16 = 2 } santa_dtype; /* q, K, V, out share it */

#define SANTA_FLAG_EMPTY_SEQ 0x1u       /* some seqlens[b] < 1: that sequence's output was zeroed  */
#define SANTA_FLAG_SYNC_TIMEOUT 0x100u  /* the single-launch step kernel gave up waiting (~0.5 s)  */
                                        /* on a unit counter: the workspace was not zero at rest   */
                                        /* (see santa_workspace_bytes); outputs are invalid        */
#define SANTA_FLAG_PEER_TIMEOUT 0x200u  /* a peer exchange gave up waiting for a rank (2 s): some   */
                                        /* rank did not make the same call; its outputs are invalid */

typedef enum {
  SANTA_PATH_AUTO = 0,        /* santa_auto_path's choice                                         */
  SANTA_PATH_STEP_KERNEL = 1, /* the single launch, mma.sync score stage (ERR_UNSUPPORTED if not eligible) */
  SANTA_PATH_TWO_KERNEL = 2,  /* score pass + PDL-chained sampler kernel                          */
  SANTA_PATH_STEP_TC = 3      /* the step kernel with its score stage on tcgen05 tensor cores    */
} santa_path;

typedef struct {
  int32_t batch;             /* B >= 1 (sequences in this call)                                 */
  int32_t n_heads;           /* H >= 1 query heads                                              */
  int32_t n_kv_heads;        /* H_kv >= 1, H % H_kv == 0, G = H/H_kv <= 8                       */
  int32_t head_dim;          /* d in {64, 128}                                                  */
  int32_t dtype;             /* santa_dtype                                                     */
  int32_t page_size;         /* P (tokens per page, multiple of 16) when paged; ignored otherwise */
  int32_t max_pages_per_seq; /* columns of page_table when paged                                */
  const int32_t* page_table; /* device int32 [batch, max_pages_per_seq] or NULL (contiguous)    */
  int32_t max_seqlen;        /* >= every seqlens[b]; sizes the workspace and the grid           */
  float scale;               /* score scale; 0 => 1/sqrt(head_dim) (Eq. 1)         */
  int32_t batch_offset;      /* global batch id of row 0 (Philox keying when sharded, sec. 8(e)) */
  int32_t head_offset;       /* global query-head id of head 0 (multiple of G when sharded)     */
} santa_geometry;

/* Human-readable name of a status code (static string, never NULL). */
const char* santa_status_string(santa_status s);

/* Library build string: version, compile target (e.g. "sm_100a") and kernel set. */
const char* santa_version(void);

/* Bytes of device workspace required by santa_decode_attention / santa_dense_reference /
 * the seq-shard phases / santa_bernoulli_scores for this geometry and budget S
 * (pure host arithmetic; returns 0 if the geometry is invalid).  The same workspace
 * may be reused across calls on one stream (one call at a time); it must be 256-byte
 * aligned and ZERO-INITIALISED ONCE before its first use: the single-launch step kernels
 * keep a launch epoch and split/exit tickets in it (tickets are zero at rest -- each is
 * reset by its last user inside the launch -- and the epoch advances once per launch), and
 * publish their cross-CTA data as words tagged with the epoch, so stale words of earlier
 * launches are never taken for current ones and no per-call memset is needed.  On a
 * workspace that was not zeroed a stale word could carry the current tag (~2^-32 per word)
 * or a poll could wait for its ~0.5 s timeout (SANTA_FLAG_SYNC_TIMEOUT) -- never a hang.
 * Everything else in it is initialised by the kernels. */
size_t santa_workspace_bytes(const santa_geometry* geo, int32_t S);

/* SANTA / S^2ANTA decode step (the north-star hot path; Eq. 4):
 * for every (b, h): s_j = (q_{b,h} . K_{b,kv(h),j}) * scale for j < seqlens[b]; p = softmax(s);
 * F = CDF of p (split-KV: per-chunk max/sum + inclusive prefix, fp64 chunk combine);
 * thresholds T_m (Philox4x32-10 stream keyed by seed, offset, global (b, h); reading #1);
 * J_m = min{j : F(j) > T_m} (reading #4); out_{b,h} = (1/S) sum_m V_{b,kv(h),J_m}.
 *   q [B,H,d], K/V per the layout above, seqlens [B] int32, S >= 1 (S > seqlen allowed:
 *   sampling is with replacement), out [B,H,d] (same dtype as q),
 *   idx_out: NULL or int32 [B,H,S] receiving J_m (token ids within the sequence).
 * Only the LOW 32 bits of `offset` enter the Philox counter.
 * Execution (santa_auto_path reports the choice): from 1024 query heads per
 * call (batch * n_heads) with S <= 256, bf16/fp16, max_seqlen <= 65536 and contiguous or
 * 128-multiple pages, the whole step is ONE cooperative persistent launch (the tcgen05 step kernel:
 * interleaved TMA score stream, score stage on tensor cores with TMEM accumulators, each
 * (b, kv-head) unit sampled as soon as its chunks are scored, chunk results published as tagged
 * words -- no fences); otherwise the split-KV score pass + a PDL-chained sampler kernel.
 * All paths draw the same thresholds; their chunk CDFs agree up to fp32/fp64 summation order and
 * their in-chunk prefixes are fp32 (two-kernel) vs 24-bit fixed point (step kernels, DESIGN.md
 * reading #23), so an index may differ between paths only where a threshold lies within ~2^-24
 * of a key boundary (the oracle-parity exemption of reading #19 covers it). */
santa_status santa_decode_attention(const santa_geometry* geo, const void* q, const void* K,
                                    const void* V, const int32_t* seqlens, int32_t S,
                                    int32_t mode, uint64_t seed, uint64_t offset, void* out,
                                    int32_t* idx_out, void* workspace, size_t workspace_bytes,
                                    void* stream);

/* Same as santa_decode_attention, and additionally records three cudaEvent_t (passed as
 * void*) on `stream`: events[0] before the score kernel, events[1] between the score
 * kernel and the sample/gather kernel, events[2] after it.  Used by bench.py to time the
 * dominant kernel inside the step (the events serialise the two launches). */
santa_status santa_decode_attention_profiled(const santa_geometry* geo, const void* q,
                                             const void* K, const void* V,
                                             const int32_t* seqlens, int32_t S, int32_t mode,
                                             uint64_t seed, uint64_t offset, void* out,
                                             int32_t* idx_out, void* workspace,
                                             size_t workspace_bytes, void* const* events,
                                             void* stream);

/* The execution path santa_decode_attention (AUTO) takes for this geometry and budget
 * (a santa_path value; -1 if the geometry is invalid).  Pure host logic. */
int32_t santa_auto_path(const santa_geometry* geo, int32_t S);

/* santa_decode_attention with an explicit execution path (santa_path: AUTO, STEP_KERNEL,
 * TWO_KERNEL, STEP_TC); AUTO is exactly santa_decode_attention.  A forced path that does not
 * support the geometry returns SANTA_ERR_UNSUPPORTED and launches nothing: the step kernels
 * (STEP_KERNEL, STEP_TC) need a bf16/fp16 cache, contiguous or pages of a multiple of 64 (STEP_TC:
 * 128) tokens, and max_seqlen <= 65536 (their sampler keeps <= 1024 chunk statistics per head in
 * registers).  Used by the tests and bench.py to compare the paths. */
santa_status santa_decode_attention_path(const santa_geometry* geo, const void* q, const void* K,
                                         const void* V, const int32_t* seqlens, int32_t S,
                                         int32_t mode, uint64_t seed, uint64_t offset, void* out,
                                         int32_t* idx_out, void* workspace,
                                         size_t workspace_bytes, int32_t path, void* stream);

/* The two phases of the two-kernel path, exposed separately (same arguments and
 * workspace; calling santa_score_phase then santa_sample_phase on one stream is exactly
 * santa_decode_attention_path(..., SANTA_PATH_TWO_KERNEL, ...)).  Phase 1 = the split-KV score pass:
 * it reads every K byte and leaves the per-chunk (m_c, l_c) and the fp32 prefix stash in
 * `workspace`.  Phase 2 = combine + thresholds + inverse CDF + gather-add (rows a3-a6). */
santa_status santa_score_phase(const santa_geometry* geo, const void* q, const void* K,
                               const int32_t* seqlens, void* workspace, size_t workspace_bytes,
                               void* stream);
santa_status santa_sample_phase(const santa_geometry* geo, const void* V, const int32_t* seqlens,
                                int32_t S, int32_t mode, uint64_t seed, uint64_t offset, void* out,
                                int32_t* idx_out, void* workspace, size_t workspace_bytes,
                                void* stream);

/* S^2ANTA-prop decode step (App. M, Algs. prop-pass1 P:1577-1594,
 * prop-budgets P:1597-1613, prop-pass2 P:1616-1641): the paper's proportional-allocation
 * estimator, a DIFFERENT (slightly biased) estimator from santa_decode_attention's global
 * samplers.  Per (b, h): tile stats m_t, l_t over tiles of B_tile = santa_prop_tile_len(geo) keys
 * (the score pass's chunks), W_t = exp(m_t - m*) l_t, quotas q_t = S W_t / Z, integer budgets
 * S_t = floor(q_t) plus one each to the S - sum floor(q_t) tiles of largest fractional part (ties
 * to the lower tile; fractional parts compared to 2^-40), then per tile systematic counts
 * c_n = floor(a0_t + p + x) - floor(a0_t + p), x = (S_t / l_t) exp(s_n - m_t), with
 * a0_t = Philox(seed, offset, tag 4, head_offset + h, batch_offset + b) draw t (reading #25);
 * out = (1/S) sum_n c_n V_n.  idx_out (optional) [B, H, S]: the emitted rows, tile-major, each
 * repeated c_n times.  Arguments, layouts, workspace and errors as santa_decode_attention (no
 * mode: the per-tile rule is systematic).  Two launches: the score pass, then the budget +
 * count + gather kernel (PDL-chained). */
santa_status santa_decode_attention_prop(const santa_geometry* geo, const void* q, const void* K,
                                         const void* V, const int32_t* seqlens, int32_t S,
                                         uint64_t seed, uint64_t offset, void* out,
                                         int32_t* idx_out, void* workspace,
                                         size_t workspace_bytes, void* stream);

/* The tile length B_tile santa_decode_attention_prop uses for this geometry (64 up to 512k
 * tokens; -1 if the geometry is invalid).  Pure host logic. */
int32_t santa_prop_tile_len(const santa_geometry* geo);

/* S^2ANTA-flash decode step (App. N, Algs. flash-mini P:1651-1667, flash-k1
 * P:1669-1689, flash-k2 P:1691-1706): uniform per-tile budgets and a deferred LSE merge -- an
 * exactly unbiased estimator that draws samples in every tile ("sample waste").  Per (b, h):
 * T = ceil(n / tile_len) tiles, S_tile = max(1, floor(S / T + 1/2)) (reading #26); in every tile
 * the systematic rows of u_n = exp(s_n - m_t) with invdelta = S_tile / l_t and
 * a0_t = Philox(seed, offset, tag 5, head_offset + h, batch_offset + b) draw t; then
 * out = (1/Z) sum_t W_t O~_t / S_tile, W_t = exp(m_t - m*) l_t, Z = sum_t W_t, O~_t = sum of the
 * tile's rows.  tile_len: a positive multiple of santa_prop_tile_len(geo) (the score pass's chunk),
 * at most 64 chunks (the paper's operating point: 256 with S = 2048 at 32k tokens);
 * otherwise SANTA_ERR_INVALID_ARG.  idx_out (optional) [B, H, M] int32 with
 * M = santa_flash_max_samples(geo, S, tile_len): the rows drawn, tile-major, -1 past the head's
 * S_tile * T; M > 16384 returns SANTA_ERR_UNSUPPORTED.  Other arguments, layouts, workspace and
 * errors as santa_decode_attention (no mode).  Two launches: the score pass, then the per-tile
 * draw + merge-weighted gather kernel (PDL-chained; the merge is folded into the gather). */
santa_status santa_decode_attention_flash(const santa_geometry* geo, const void* q, const void* K,
                                          const void* V, const int32_t* seqlens, int32_t S,
                                          int32_t tile_len, uint64_t seed, uint64_t offset, void* out,
                                          int32_t* idx_out, void* workspace, size_t workspace_bytes,
                                          void* stream);

/* Row length M of santa_decode_attention_flash's idx_out: the largest S_tile * T over sequence
 * lengths <= geo->max_seqlen (-1 if the geometry, S or tile_len is invalid).  Pure host logic. */
int32_t santa_flash_max_samples(const santa_geometry* geo, int32_t S, int32_t tile_len);

/* Exact dense decode attention softmax(q K^T * scale) V (Eq. 1) with the same
 * split-KV score pass and a flash-decoding LSE combine; the in-repo reference the SANTA
 * latency is reported against.  Arguments as above. */
santa_status santa_dense_reference(const santa_geometry* geo, const void* q, const void* K,
                                   const void* V, const int32_t* seqlens, void* out,
                                   void* workspace, size_t workspace_bytes, void* stream);

/* Bernoulli qK^T score stage (Eq. 5; Eq. 6; App. C), reading only
 * the selected feature rows of a FEATURE-MAJOR key cache Kt:
 *   contiguous Kt [B, H_kv, d, max_seqlen]; paged pool [num_pages, H_kv, d, page_size].
 * mean_group = 1: per (b, kv-head) m_i = mean_g |q_{g,i}|, norm = max_i m_i, counts c_i of
 *   B draws of Bernoulli(m_i/norm) (stratified: floor(B a) + 1[u < frac(B a)], reading #11;
 *   standard: #{n : u_{i,n} < a_i}); p_hat_g = sum_{c_i>0} (norm c_i / B) q_{g,i}/m_i Kt_i.
 * mean_group = 0: per-head ternary estimator p_hat = (norm/B) sum_i c_i sign(q_i) Kt_i.
 * Writes scores [B, H, max_seqlen] fp32 = scale * p_hat (0 at positions >= seqlens[b]) and,
 * if feature_mask != NULL, uint8 [B, H_kv (mean_group) or H, d] = 1 for fetched features.
 * Philox tags 3 (mean-group, keyed by global kv-head) / 2 (per head), reading #1. */
santa_status santa_bernoulli_scores(const santa_geometry* geo, const void* q, const void* Kt,
                                    const int32_t* seqlens, int32_t B, int32_t stratified,
                                    int32_t mean_group, uint64_t seed, uint64_t offset,
                                    float* scores, uint8_t* feature_mask, void* workspace,
                                    size_t workspace_bytes, void* stream);

/* Config 5: Bernoulli score stage + S^2ANTA value stage: scores from
 * santa_bernoulli_scores (kept in the workspace), then softmax -> sampling -> gather-add
 * of V exactly as santa_decode_attention.  Bernoulli draws use (seed, offset) with tags
 * 2/3; the value sampler uses the same (seed, offset) with tag 1. */
santa_status santa_decode_attention_bernoulli(const santa_geometry* geo, const void* q,
                                              const void* Kt, const void* V,
                                              const int32_t* seqlens, int32_t B,
                                              int32_t stratified, int32_t mean_group, int32_t S,
                                              int32_t mode, uint64_t seed, uint64_t offset,
                                              void* out, int32_t* idx_out, void* workspace,
                                              size_t workspace_bytes, void* stream);

/* Sequence sharding, phase 1 (config 4; reading #18).  `geo` describes THIS rank's
 * shard: K_shard holds the shard's tokens at positions 0..shard_seqlens[b]-1.  Runs the
 * split-KV score pass on the shard and reduces it to per-(b, h) statistics
 *   stats_out[b,h,0] = m_r  = max_j s_j * log2(e)            (fp64; -inf if empty)
 *   stats_out[b,h,1] = L_r  = sum_j 2^(s_j log2(e) - m_r)     (fp64; 0 if empty)
 * stats_out is device fp64 [B, H, 2].  The per-chunk statistics and prefix stash stay in
 * `workspace` for phase 2, which must use the same workspace. */
santa_status santa_seqshard_stats(const santa_geometry* geo, const void* q, const void* K_shard,
                                  const int32_t* shard_seqlens, double* stats_out,
                                  void* workspace, size_t workspace_bytes, void* stream);

/* Sequence sharding, phase 2.  stats_all is device fp64 [world, B, H, 2]: every rank's
 * phase-1 stats (all-gathered by the caller over NCCL).  Every rank forms the identical
 * global shard CDF F_r = sum_{r'<=r} 2^(m_r'-m*) L_r' / Z, draws the identical global
 * thresholds T_m, keeps the strata with F_{rank-1} <= T_m < F_rank and samples them in its
 * shard.  Writes partial_out [B, H, d] fp32 = (1/S) sum_{own m} V_{J_m} (zero if none),
 * to be SUM-reduced across ranks by the caller, and, if idx_out != NULL, int32 [B, H, S]
 * with the GLOBAL token id (token_offset[b] + local id) for owned strata and -1 elsewhere.
 * token_offset: device int32 [B], this shard's first global token id per sequence. */
santa_status santa_seqshard_sample_gather(const santa_geometry* geo, const double* stats_all,
                                          int32_t rank, int32_t world,
                                          const int32_t* token_offset, const void* V_shard,
                                          const int32_t* shard_seqlens, int32_t S, int32_t mode,
                                          uint64_t seed, uint64_t offset, float* partial_out,
                                          int32_t* idx_out, void* workspace,
                                          size_t workspace_bytes, void* stream);

/* End-to-end decode step through HOST buffers (used for bench.py's "e2e"): copies q_host
 * [B,H,d] and the current token's k_new_host / v_new_host [B,H_kv,d] (pinned host memory)
 * into the device staging buffers q_dev / k_new_dev / v_new_dev, appends k_new / v_new to
 * the cache at position seqlens[b]-1 (the "+1 slot"), runs
 * santa_decode_attention into out_dev and copies it to out_host; synchronises `stream`
 * before returning.  Every check of santa_decode_attention runs BEFORE the first copy or launch,
 * so an invalid call leaves the cache untouched.
 * Bytes moved per call: H2D (B*H + 2*B*H_kv)*d*e, D2H B*H*d*e. */
santa_status santa_decode_step_host(const santa_geometry* geo, const void* q_host,
                                    const void* k_new_host, const void* v_new_host,
                                    void* q_dev, void* k_new_dev, void* v_new_dev, void* K,
                                    void* V, const int32_t* seqlens, int32_t S, int32_t mode,
                                    uint64_t seed, uint64_t offset, void* out_dev,
                                    void* out_host, void* workspace, size_t workspace_bytes,
                                    void* stream);

/* As santa_decode_step_host with ONE packed host buffer and an optional sync -- the form a
 * serving loop uses: qkv_host (pinned) = [q (B*H*d) | k_new (B*H_kv*d) | v_new (B*H_kv*d)]
 * elements of the geometry's dtype, copied with one H2D into the device staging buffer qkv_dev
 * (same size), then the KV append, santa_decode_attention, and one D2H of out_dev into out_host
 * (pinned, B*H*d).  synchronize != 0: syncs `stream` before returning (out_host is valid);
 * synchronize == 0: fully asynchronous, out_host is valid once the caller syncs the stream.
 * Zero copy: a 16-B aligned PAGE-LOCKED qkv_host (cudaHostAlloc / cudaHostRegister) is read by the
 * staging kernel itself (q rows -> qkv_dev, k/v rows -> the cache) and a page-locked out_host is
 * written by the decode kernels themselves (out_dev then unused) -- no copy-engine transfers;
 * pageable buffers use cudaMemcpyAsync.  All argument checks run before the first copy or launch
 * (an invalid call leaves the cache untouched).  The host must not modify qkv_host / read out_host
 * before the stream reaches the end of this call's work.  A page-locked qkv_host must hold the step's
 * inputs when the call is made: the staging kernel is launched with programmatic dependent launch and
 * reads it BEFORE the preceding kernel in the stream has finished (its device writes -- q staging, the
 * cache slot -- wait for that kernel), so it must not be produced by GPU work still in flight.
 * Bytes moved per call: H2D (B*H + 2*B*H_kv)*d*e, D2H B*H*d*e. */
santa_status santa_decode_step_host_packed(const santa_geometry* geo, const void* qkv_host, void* qkv_dev,
                                           void* K, void* V, const int32_t* seqlens, int32_t S,
                                           int32_t mode, uint64_t seed, uint64_t offset, void* out_dev,
                                           void* out_host, void* workspace, size_t workspace_bytes,
                                           int32_t synchronize, void* stream);

/* Decode-loop integration.
 *
 * santa_decode_attention_append: the decode step WITH the KV append of the current token, the way
 * FA-2's decode kernel appends: k_new / v_new are device [batch, n_kv_heads,
 * head_dim] rows (dtype of the cache, 16-B aligned) written into K / V (now writable) at slot
 * seqlens[b] - 1 (seqlens include the new token, reading #10), then the step of
 * santa_decode_attention.  On the two-kernel path (AUTO below 1024 query heads) the append is fused
 * into the score pass: the TMA producer lane that streams the stage holding the slot writes both
 * rows first (then a generic->async proxy fence, so its own TMA load sees the new key); on the
 * single-launch step kernels and the fp32 / odd-page fallback a one-CTA-per-(b, kv head) append
 * kernel runs first.  Same validation, errors and determinism as santa_decode_attention (nothing
 * is written on error).
 *
 * Per-layer budgets (App. K: a learned schedule assigns each transformer layer its own
 * S under a global budget): santa_layer_schedule is a HOST array S[n_layers] (each >= 1, <= 4096).
 * santa_decode_attention_layer decodes layer `layer` with S = sched->S[layer] and the Philox
 * offset (offset * n_layers + layer), so every (step, layer) has its own stream; k_new / v_new
 * may be NULL (no append) or the new token's rows (append as above).  idx_out rows are
 * sched->S[layer] long.  santa_schedule_workspace_bytes = the workspace for every layer of the
 * schedule (the max over its S; one workspace serves all layers of a stream in turn). */
typedef struct santa_layer_schedule {
  int32_t n_layers;
  const int32_t* S; /* host [n_layers] */
} santa_layer_schedule;

santa_status santa_decode_attention_append(const santa_geometry* geo, const void* q, void* K, void* V,
                                           const void* k_new, const void* v_new, const int32_t* seqlens,
                                           int32_t S, int32_t mode, uint64_t seed, uint64_t offset, void* out,
                                           int32_t* idx_out, void* workspace, size_t workspace_bytes,
                                           void* stream);
size_t santa_schedule_workspace_bytes(const santa_geometry* geo, const santa_layer_schedule* sched);
santa_status santa_decode_attention_layer(const santa_geometry* geo, const santa_layer_schedule* sched,
                                          int32_t layer, const void* q, void* K, void* V, const void* k_new,
                                          const void* v_new, const int32_t* seqlens, int32_t mode,
                                          uint64_t seed, uint64_t offset, void* out, int32_t* idx_out,
                                          void* workspace, size_t workspace_bytes, void* stream);

/* Device Philox4x32-10 uniforms for testing the device RNG against the Random123 KAT and
 * the oracle stream: out[i] = u(draw i) of the stream (seed, offset, tag, h_global, b_global),
 * u = r * 2^-32 (reading #1).  out is device fp64 [n]; if raw_out != NULL it receives the 4
 * raw words of block 0 for ctr=(ctr0..3), key=(key0,key1) (KAT check). */
santa_status santa_philox_uniforms(uint64_t seed, uint64_t offset, int32_t tag, int32_t h_global,
                                   int32_t b_global, int32_t n, double* out, const uint32_t* ctr_key_host,
                                   uint32_t* raw_out, void* stream);

/* Reads (and clears) the workspace flag word: syncs `stream`, copies it to *flags_out. */
santa_status santa_read_error_flags(void* workspace, uint32_t* flags_out, void* stream);

/* Peer-memory exchange for the sequence-sharded step (config 4).
 *
 * The two collectives of santa_seqshard_* -- the all-gather of every rank's [B, H, 2] fp64
 * (m_r, L_r) and the SUM of the [B, H, d] fp32 partial outputs (reading #18; the exchange is an
 * extension, no paper passage) -- as ONE kernel each over NVLink peer memory: every rank stores
 * its payload into slot `rank` of every rank's exchange buffer (P2P stores through CUDA-IPC
 * mappings), releases a per-(source, block) flag there, acquires the flags of all sources in its
 * own buffer and consumes its slots.  The SUM adds the slots in rank order 0..world-1 in fp32,
 * so every rank gets bit-identical results.
 *
 * group->bufs[r] is rank r's exchange buffer as addressable from THIS process (its own
 * allocation for r == rank, a santa_ipc_import mapping otherwise), every one 256-B aligned and
 * group->buf_bytes long (>= santa_peer_buffer_bytes(world, largest payload)), zeroed by the
 * caller once before the first call (flag word at offset 0 readable with santa_read_error_flags).
 * `epoch` numbers the calls on the group: 1, 2, 3, ... (+1 per call, all ranks the same sequence
 * of calls); call e uses buffer half e & 1.
 *
 * n_local ranks are served by one launch: ranks[l], src[l], dst[l] (host arrays of device
 * pointers) for l < n_local.  A multi-GPU run passes n_local = 1 (its own rank).  n_local = world
 * emulates the whole group in ONE cooperative launch on one GPU (every rank's buffer allocated on
 * it) -- the test configuration; separate per-rank launches that wait on each other on one GPU
 * are not supported.  A wait that sees no flag for 2 s gives up and sets SANTA_FLAG_PEER_TIMEOUT in
 * the own buffer's flag word (never a hang).
 *
 * allgather: src[l] = `bytes` (multiple of 16) of payload; dst[l] = [world][bytes].
 * allreduce_f32: src[l], dst[l] = `count` fp32 (count * 4 a multiple of 16); dst may equal src.
 * Errors: SANTA_ERR_INVALID_ARG (NULL, world not in 1..8, ranks repeated / out of range,
 * epoch 0), SANTA_ERR_ALIGNMENT, SANTA_ERR_WORKSPACE (payload larger than a slot),
 * SANTA_ERR_CUDA (launch refused). */
typedef struct {
  int32_t world;      /* ranks in the group, 1..8 */
  void* bufs[8];      /* bufs[r]: rank r's exchange buffer, mapped into this process */
  size_t buf_bytes;   /* bytes of every rank's buffer */
} santa_peer_group;

#define SANTA_IPC_HANDLE_BYTES 64

/* Buffer bytes for payloads of up to max_payload_bytes per rank (0 if world not in 1..8). */
size_t santa_peer_buffer_bytes(int32_t world, size_t max_payload_bytes);
santa_status santa_peer_allgather(const santa_peer_group* group, int32_t n_local, const int32_t* ranks,
                                  const void* const* src, void* const* dst, size_t bytes, uint32_t epoch,
                                  void* stream);
santa_status santa_peer_allreduce_f32(const santa_peer_group* group, int32_t n_local, const int32_t* ranks,
                                      const float* const* src, float* const* dst, size_t count, uint32_t epoch,
                                      void* stream);

/* CUDA-IPC plumbing for the exchange buffers (host only, no kernel): santa_ipc_export writes the
 * 64-B handle of the allocation holding dev_ptr and dev_ptr's offset in it; santa_ipc_import (in
 * another process) maps it and returns the peer's dev_ptr (base + offset) and the mapping base,
 * which santa_ipc_close unmaps.  An allocation cannot be imported into the process that exported
 * it (pass the own pointer instead). */
santa_status santa_ipc_export(const void* dev_ptr, void* handle_out, size_t* offset_out);
santa_status santa_ipc_import(const void* handle, size_t offset, void** dev_ptr_out, void** base_out);
santa_status santa_ipc_close(void* base);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif

#ifdef __cplusplus
}
#endif
#endif /* SANTA_H_ */
