// runners.cuh -- the launchers of every kernel family (declared in host.cuh).  Included only by
// inst.cu, which instantiates them for one (family, dtype, head_dim) per object file.
#pragma once
#include "host.cuh"

namespace santa_host {

template <typename T, int D, int G>
santa_status RunScore<T, D, G>::run(const DecodeArgs& a) {
  ScoreParams p = make_score_params(a);
  if (a.events) cudaEventRecord(a.events[0], a.st);
  const bool stream = !a.g->page_table || a.g->page_size % kStageKeys == 0;
  if constexpr (sizeof(T) == 2) if (stream) {
    CUtensorMap tm;
    const uint64_t rows = a.g->page_table ? (uint64_t)0x7fffffff
                                          : (uint64_t)a.g->batch * a.g->n_kv_heads * a.g->max_seqlen;
    if (!make_kmap(&tm, a.K, rows, D, a.g->dtype)) return SANTA_ERR_CUDA;
    constexpr size_t kStageBytes = (D / 64) * 8192;
    constexpr int NW = kStreamWarps, SPW = kStreamSlots;
    const size_t smem = 1024 + (size_t)NW * G * p.L * 4 + (size_t)NW * SPW * (kStageBytes + 16);
    if (smem <= 220 * 1024) {  // else: per-warp score buffers too large (G * L big) -> fallback kernel
    const int total = a.g->batch * a.g->n_kv_heads * p.Cmax;
    const int grid = total < num_sms() * SANTA_STREAM_CTAS ? total : num_sms() * SANTA_STREAM_CTAS;
    if (a.k_new) {  // the fused KV append (santa_decode_attention_append)
      auto kern = score_stream_append_kernel<T, D, G, NW, SPW>;
      if (ensure_smem(kern, smem) != cudaSuccess) return SANTA_ERR_CUDA;
      const AppendParams ap{a.k_new, a.v_new, a.K_w, a.V_w};
      if (launch(kern, dim3(grid), dim3(32 * (NW + 1)), smem, a.st, true, tm, p, ap) != cudaSuccess)
        return SANTA_ERR_CUDA;
      return SANTA_OK;
    }
    auto kern = score_stream_kernel<T, D, G, NW, SPW>;
    if (ensure_smem(kern, smem) != cudaSuccess) return SANTA_ERR_CUDA;
    static const bool no_pdl = std::getenv("SANTA_SCORE_NO_PDL") != nullptr;  // A/B switch (tools)
    if (launch(kern, dim3(grid), dim3(32 * (NW + 1)), smem, a.st, a.events == nullptr && !no_pdl, tm, p) !=
        cudaSuccess)
      return SANTA_ERR_CUDA;
    return SANTA_OK;
    }
  }
  {
    dim3 grid(a.L.Cmax, a.g->n_kv_heads, a.g->batch);
    const size_t smem = (size_t)G * p.L * 4;
    if (ensure_smem(score_chunk_kernel<T, D, G>, smem) != cudaSuccess) return SANTA_ERR_CUDA;
    if (launch(score_chunk_kernel<T, D, G>, grid, dim3(128), smem, a.st, false, p) != cudaSuccess)
      return SANTA_ERR_CUDA;
  }
  return SANTA_OK;
}

template <typename T, int D, int G>
santa_status RunSample<T, D, G>::run(const DecodeArgs& a) {
  SampleParams p = make_sample_params(a);
  // the low-latency sampler (sample_fast.cuh) when its grid is one wave (its CTAs hold one SM each);
  // beyond that the 256-thread cluster sampler below is faster (config 5, batch 16: 61 vs ~33 us)
  const int heads = a.g->batch * a.g->n_heads;
  if (p.L == 64 && a.stats_all == nullptr && heads <= num_sms()) {
    // CTAs per head: up to a 4-CTA cluster while the grid stays one wave (config 2: 32 heads x 4;
    // tools/tail_sweep.py: CS = 1 / 2 / 4 -> 26.8 / 24.6 / 22.6 us per step), >= 8 strata per CTA
    // (whole 64-strata super-blocks per CTA: the summation tree, hence the output bits, do not depend
    // on CS -- batch x kv-head slabs of any size give the same bits)
    int CS = 1;
    while (CS < 4 && heads * CS * 2 <= num_sms() && CS * 2 * 64 <= a.S) CS *= 2;
    p.cluster = CS;
    const size_t smem = sample_fast_smem_bytes(p.Cmax, D, CS, a.S);
    if (ensure_smem(sample_fast_kernel<T, D, G>, smem) != cudaSuccess) return SANTA_ERR_CUDA;
    if (a.events) cudaEventRecord(a.events[1], a.st);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(a.g->n_heads * CS, a.g->batch);
    cfg.blockDim = dim3(kFastThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = a.st;
    cudaLaunchAttribute attr[2];
    int na = 0;
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = CS;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
    if (a.events == nullptr) {
      attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[na].val.programmaticStreamSerializationAllowed = 1;
      ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    if (cudaLaunchKernelEx(&cfg, sample_fast_kernel<T, D, G>, p) != cudaSuccess) return SANTA_ERR_CUDA;
    if (a.events) cudaEventRecord(a.events[2], a.st);
    return SANTA_OK;
  }
  // CTAs per head: a thread-block cluster of CS CTAs splits the S strata (more SMs on the
  // latency-bound search/gather), partials summed through DSMEM.  Aim at >= ~2 CTAs per SM.
  int CS = 1;
  while (CS < 4 && heads * CS * 2 <= 2 * num_sms() && CS * 2 <= a.S) CS *= 2;
  p.cluster = CS;
  const size_t smem = sample_smem_bytes(p.Cmax, (a.S + CS - 1) / CS, D, kSampleThreads);
  // more than two CTAs per SM needed for one wave: the 4-per-SM build (64 registers, 4 samples in
  // flight per half-warp) -- config 5 (512 heads): see DESIGN.md sec. 5
  static const int variant = std::getenv("SANTA_SAMPLE_MINB") ? std::atoi(std::getenv("SANTA_SAMPLE_MINB")) : 0;
  const long ctas = (long)heads * CS;
  const bool occ4 = variant == 4 || (variant == 0 && ctas > 2L * num_sms() && smem * 4 <= 200 * 1024);
  auto kern = occ4 ? sample_gather_kernel<T, D, G, 4> : sample_gather_kernel<T, D, G, 1>;
  if (ensure_smem(kern, smem) != cudaSuccess) return SANTA_ERR_CUDA;
  if (a.events) cudaEventRecord(a.events[1], a.st);
  const bool pdl = a.events == nullptr && a.stats_all == nullptr;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(a.g->n_heads * CS, a.g->batch);
  cfg.blockDim = dim3(kSampleThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = a.st;
  cudaLaunchAttribute attr[2];
  int na = 0;
  attr[na].id = cudaLaunchAttributeClusterDimension;
  attr[na].val.clusterDim.x = CS;
  attr[na].val.clusterDim.y = 1;
  attr[na].val.clusterDim.z = 1;
  ++na;
  if (pdl) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  if (cudaLaunchKernelEx(&cfg, kern, p) != cudaSuccess) return SANTA_ERR_CUDA;
  if (a.events) cudaEventRecord(a.events[2], a.st);
  return SANTA_OK;
}

template <typename T, int D, int G>
santa_status RunProp<T, D, G>::run(const DecodeArgs& a) {
  SampleParams p = make_sample_params(a);
  int CS = 1;
  const int heads = a.g->batch * a.g->n_heads;
  while (CS < 4 && heads * CS * 2 <= 2 * num_sms() && CS * 2 <= a.S) CS *= 2;
  p.cluster = CS;
  const size_t smem = prop_smem_bytes(p.Cmax, (a.S + CS - 1) / CS, D, kSampleThreads);
  if (smem > 227 * 1024) return SANTA_ERR_UNSUPPORTED;
  if (ensure_smem(prop_gather_kernel<T, D, G>, smem) != cudaSuccess) return SANTA_ERR_CUDA;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(a.g->n_heads * CS, a.g->batch);
  cfg.blockDim = dim3(kSampleThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = a.st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CS;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  if (cudaLaunchKernelEx(&cfg, prop_gather_kernel<T, D, G>, p) != cudaSuccess) return SANTA_ERR_CUDA;
  return SANTA_OK;
}

template <typename T, int D, int G>
santa_status RunFlash<T, D, G>::run(const DecodeArgs& a, int cpt, int mmax) {
  SampleParams p = make_sample_params(a);
  int CS = 1;
  const int heads = a.g->batch * a.g->n_heads;
  // up to 4 CTAs per head within one wave (8-CTA clusters measured slower: 132 registers x 256
  // threads fit one CTA per SM, so 256 CTAs ran in two waves)
  while (CS < 4 && heads * CS * 2 <= 2 * num_sms() && CS * 2 <= mmax) CS *= 2;
  p.cluster = CS;
  const size_t smem = flash_smem_bytes(p.Cmax, cpt, (mmax + CS - 1) / CS, D, kSampleThreads);
  if (smem > 227 * 1024) return SANTA_ERR_UNSUPPORTED;
  if (ensure_smem(flash_gather_kernel<T, D, G>, smem) != cudaSuccess) return SANTA_ERR_CUDA;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(a.g->n_heads * CS, a.g->batch);
  cfg.blockDim = dim3(kSampleThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = a.st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CS;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  if (cudaLaunchKernelEx(&cfg, flash_gather_kernel<T, D, G>, p, cpt, mmax) != cudaSuccess) return SANTA_ERR_CUDA;
  return SANTA_OK;
}

// the tensor-core variant (santa_step_tc_kernel): 128-key tiles, pages of a multiple of 128
template <typename T, int D, int G>
santa_status RunStep<T, D, G>::run_tc(const DecodeArgs& a, const ScoreParams& sp, const SampleParams& pp, int CS, int grid) {
  if constexpr (sizeof(T) != 2) {
    return SANTA_ERR_UNSUPPORTED;
  } else {
    constexpr int NSW = kStepSamplers, NT = 32 * kTcWarps;
    if (a.g->page_table && a.g->page_size % kTcTileKeys != 0) return SANTA_ERR_UNSUPPORTED;
    const size_t smem = step_tc_score_smem_bytes(D, G) + step_sample_smem_bytes(pp.Cmax, (a.S + CS - 1) / CS, D);
    if (smem > 226 * 1024) return SANTA_ERR_UNSUPPORTED;
    auto kern = santa_step_tc_kernel<T, D, G, NSW>;
    if (ensure_smem(kern, smem) != cudaSuccess) return SANTA_ERR_CUDA;
    if (!fits_one_per_sm(kern, NT, smem)) return SANTA_ERR_UNSUPPORTED;
    CUtensorMap tk, tq;
    const uint64_t rows = a.g->page_table ? (uint64_t)0x7fffffff
                                          : (uint64_t)a.g->batch * a.g->n_kv_heads * a.g->max_seqlen;
    if (!make_kmap(&tk, a.K, rows, D, a.g->dtype, 64)) return SANTA_ERR_UNSUPPORTED;
    if (!make_qmap(&tq, a.q, (uint64_t)a.g->batch * a.g->n_heads, D, a.g->dtype, G)) return SANTA_ERR_UNSUPPORTED;
    StepSync sy = make_step_sync(a);
    SampleParams pq = pp;
    pq.cluster = CS;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(NT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = a.st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return coop_status(cudaLaunchKernelEx(&cfg, kern, tk, tq, sp, pq, sy));
  }
}

template <typename T, int D, int G>
santa_status RunStep<T, D, G>::run(const DecodeArgs& a) {
  if constexpr (sizeof(T) != 2) {
    return SANTA_ERR_UNSUPPORTED;
  } else {
    if (!stream_eligible(a.g) || a.L.L != kStepStageKeys) return SANTA_ERR_UNSUPPORTED;
    // the sampler group's chunk-CDF registers hold <= kStepMaxChunks chunks (65,536 tokens)
    if (a.L.Cmax > kStepMaxChunks) return SANTA_ERR_UNSUPPORTED;
    constexpr int NW = kStepConsumers, SPW = kStepSlots, NSW = kStepSamplers, NT = 32 * (NW + 1 + NSW);
    ScoreParams sp = make_score_params(a);
    SampleParams pp = make_sample_params(a);
    // splits per head: aim at one sampler round (<= 64 strata) per item, so the exposed tail (the
    // last unit's items) is one gather round, but keep the total at <= 4 items per CTA: every item
    // repeats the chunk-CDF combine, and at large batch the sampler work must stay hidden under
    // the stream (config 3, S = 512: 8192 items -> 661 us vs 1024 items -> see DESIGN.md sec. 5)
    const int grid = num_sms(), heads = a.g->batch * a.g->n_heads;
    int CS = 1;
    while (CS * 2 <= kStepMaxSplits && CS * 64 < a.S && heads * CS * 2 <= 4 * grid) CS *= 2;
    pp.cluster = CS;
    if (a.tensor_core) return run_tc(a, sp, pp, CS, grid);
    const size_t smem = step_score_smem_bytes(D, G, NW, SPW) + step_sample_smem_bytes(pp.Cmax, (a.S + CS - 1) / CS, D);
    if (smem > 226 * 1024) return SANTA_ERR_UNSUPPORTED;  // 227 KiB per CTA minus static smem
    auto kern = santa_step_kernel<T, D, G, NW, SPW, NSW>;
    if (ensure_smem(kern, smem) != cudaSuccess) return SANTA_ERR_CUDA;
    if (!fits_one_per_sm(kern, NT, smem)) return SANTA_ERR_UNSUPPORTED;
    CUtensorMap tm;
    const uint64_t rows = a.g->page_table ? (uint64_t)0x7fffffff
                                          : (uint64_t)a.g->batch * a.g->n_kv_heads * a.g->max_seqlen;
    if (!make_kmap(&tm, a.K, rows, D, a.g->dtype, kStepStageKeys)) return SANTA_ERR_UNSUPPORTED;
    StepSync sy = make_step_sync(a);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(NT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = a.st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return coop_status(cudaLaunchKernelEx(&cfg, kern, tm, sp, pp, sy));
  }
}

template <typename T, int D, int G, int NW, int SPW>
santa_status run_dense_split(const DecodeArgs& a, const DenseParams& p) {
  constexpr size_t kStageBytes = 2 * (D / 64) * kDenseStageKeys * 128;
  const size_t smem = 1024 + (size_t)NW * SPW * (kStageBytes + 16) + (size_t)NW * 8 * kPRow * 2;
  auto kern = dense_split_kernel<T, D, G, NW, SPW>;
  if (ensure_smem(kern, smem) != cudaSuccess) return SANTA_ERR_CUDA;
  CUtensorMap tk, tv;
  const uint64_t rows = a.g->page_table ? (uint64_t)0x7fffffff
                                        : (uint64_t)a.g->batch * a.g->n_kv_heads * a.g->max_seqlen;
  if (!make_kmap(&tk, a.K, rows, D, a.g->dtype, kDenseStageKeys) ||
      !make_kmap(&tv, a.V, rows, D, a.g->dtype, kDenseStageKeys))
    return SANTA_ERR_CUDA;
  DenseSplitParams dp;
  dp.q = a.q;
  dp.kv = p.kv;
  dp.seqlens = a.seqlens;
  dp.B = p.B;
  dp.H = p.H;
  dp.Hkv = p.Hkv;
  dp.scale_log2 = p.scale_log2;
  dp.part_o = at<float>(a.ws, a.L.dense_o);
  dp.part_ml = at<float2>(a.ws, a.L.dense_ml);
  dp.out = a.out;
  dp.flags = p.flags;
  const int grid = std::min(num_sms(), kDenseSplitMaxCtas);
  if (launch(kern, dim3(grid), dim3(32 * (NW + 1)), smem, a.st, true, tk, tv, dp) != cudaSuccess)
    return SANTA_ERR_CUDA;
  // slots per head ~ (CTAs per unit + 1) x NW: 16 parts per output coordinate when that is large
  // (config 2: ~19 CTAs per unit -> one L2 round trip), else one 4-part CTA per head (config 3)
  const int units = a.g->batch * a.g->n_kv_heads;
  const bool many = (grid / units + 1) * NW >= 32;
  constexpr int NPB = 16, NPS = kDenseCombineThreads / D;  // NPS: one CTA per head
  const cudaError_t e =
      many ? launch(dense_split_combine<T, D, G, NW, NPB>, dim3(a.g->n_heads * (D * NPB / kDenseCombineThreads),
                                                                  a.g->batch),
                    dim3(kDenseCombineThreads), 0, a.st, true, dp, grid)
           : launch(dense_split_combine<T, D, G, NW, NPS>, dim3(a.g->n_heads * (D * NPS / kDenseCombineThreads),
                                                                  a.g->batch),
                    dim3(kDenseCombineThreads), 0, a.st, true, dp, grid);
  if (e != cudaSuccess) return SANTA_ERR_CUDA;
  return SANTA_OK;
}

template <typename T, int D, int G>
santa_status RunDense<T, D, G>::run(const DecodeArgs& a) {
  DenseParams p;
  p.q = a.q;
  p.K = a.K;
  p.V = a.V;
  p.kv = kv_layout(a.g);
  p.seqlens = a.seqlens;
  p.B = a.g->batch;
  p.H = a.g->n_heads;
  p.Hkv = a.g->n_kv_heads;
  p.scale_log2 = scale_log2(a.g);
  p.cstats = at<float2>(a.ws, a.L.cstats);
  p.opart = at<float>(a.ws, a.L.stash);
  p.Cmax = a.L.Cmax256;
  p.out = a.out;
  p.flags = at<uint32_t>(a.ws, a.L.flags);
  bool done = false;
  if constexpr (sizeof(T) == 2) {
    if (stream_eligible(a.g)) {  // balanced split-KV tensor-core kernel + its LSE combine
      // warps x slots by the bytes each SM streams: 3 x 4 below ~4 MiB per SM (config 2: 28.0 vs 29.7
      // us for 6 x 2 -- fewer partials to merge), 5 x 2 above (config 3, 4 GiB: 631 vs 672 us for 6 x 2)
      const double per_sm = 2.0 * a.g->batch * a.g->n_kv_heads * (double)a.g->max_seqlen * D * sizeof(T) / num_sms();
      return per_sm < 4.0 * (1 << 20) ? run_dense_split<T, D, G, kDenseWarps, kDenseSlots>(a, p)
                                      : run_dense_split<T, D, G, kDenseWarpsLarge, kDenseSlotsLarge>(a, p);
    }
  }
  if (!done) {
    dim3 grid(a.L.Cmax256, a.g->n_kv_heads, a.g->batch);
    if (launch(dense_partial_kernel<T, D, G>, grid, dim3(kScoreThreads), 0, a.st, false, p) != cudaSuccess)
      return SANTA_ERR_CUDA;
  }
  if (launch(dense_combine_kernel<T, D>, dim3(a.g->n_heads, a.g->batch), dim3(256), 0, a.st, true, p) !=
      cudaSuccess)
    return SANTA_ERR_CUDA;
  return SANTA_OK;
}

// mode 0: standalone scores (scores != NULL, no stash); mode 1: fused into the decode step
template <typename T, int D, int G>
santa_status RunBern<T, D, G>::run(const DecodeArgs& a, const void* Kt, int nB, int stratified, int mean_group,
                        float* scores, uint8_t* mask, bool for_decode) {
  BernParams p = {};
  p.q = a.q;
  p.Kt = Kt;
  p.seqlens = a.seqlens;
  p.B = a.g->batch;
  p.H = a.g->n_heads;
  p.Hkv = a.g->n_kv_heads;
  p.nB = nB;
  p.stratified = stratified;
  p.mean_group = mean_group;
  p.seed = a.seed;
  p.offset = a.offset;
  p.batch_offset = a.g->batch_offset;
  p.head_offset = a.g->head_offset;
  p.scale = a.g->scale > 0.f ? a.g->scale : 1.0f / std::sqrt((float)D);
  char* bern = at<char>(a.ws, a.L.bern);
  const size_t units = (size_t)a.g->batch * a.g->n_kv_heads;
  p.w = reinterpret_cast<float*>(bern);
  p.sel = reinterpret_cast<int*>(bern + units * G * D * 4);
  p.sel_n = reinterpret_cast<int*>(bern + units * G * D * 4 + units * D * 4);
  p.feature_mask = mask;
  p.page_table = a.g->page_table;
  p.page_size = a.g->page_size;
  p.max_pages = a.g->max_pages_per_seq;
  p.scores = scores;
  p.score_stride = a.g->max_seqlen;
  p.stash = for_decode ? at<float>(a.ws, a.L.stash) : nullptr;
  p.cstats = at<float2>(a.ws, a.L.cstats);
  // decode: 64-key stats/stash in the standard layout when L = 64 (the sampler's fast ballot
  // search), else per 256-key chunk
  p.sub64 = (for_decode && a.L.L == 64) ? 1 : 0;
  p.Cmax = p.sub64 ? a.L.Cmax : a.L.Cmax256;
  p.stash_stride = p.sub64 ? a.L.Cmax * 64 : a.L.Cmax256 * kDenseChunk;
  p.tickets = at<uint32_t>(a.ws, a.L.tickets);
  p.flags = at<uint32_t>(a.ws, a.L.flags);
  // bf16 decode on 64-key chunks with 16-B aligned feature rows: the TMA + tensor-core stream
  // (bern_tma_kernel.cuh); its B fragments are built by the weights kernel
  static const bool force_fma = std::getenv("SANTA_BERN_FMA") != nullptr;  // A/B switch (tools)
  bool tma = false;
  if constexpr (std::is_same<T, __nv_bfloat16>::value) {
    const int P = a.g->page_table ? a.g->page_size : a.g->max_seqlen;
    tma = for_decode && p.sub64 && scores == nullptr && P % 8 == 0 && (reinterpret_cast<uintptr_t>(Kt) & 15) == 0 &&
          (a.g->page_table == nullptr || P % kBtKeys == 0 || (P >= kBtMinPage && kBtKeys % P == 0)) &&
          !force_fma;
  }
  p.wfrag = tma ? at<uint2>(a.ws, a.L.bfrag) : nullptr;
  if (launch(bern_weights_kernel<T, D, G>, dim3(a.g->n_kv_heads, a.g->batch), dim3(D), 0, a.st, true, p) !=
      cudaSuccess)
    return SANTA_ERR_CUDA;
  if constexpr (std::is_same<T, __nv_bfloat16>::value) {
    if (tma) {
      const int nblk = (a.g->max_seqlen + kBtKeys - 1) / kBtKeys;
      const int items = a.g->batch * a.g->n_kv_heads * nblk;
      const int grid = std::min(items, num_sms());
      const size_t smem = bern_tma_smem_bytes(G);
      if (ensure_smem(bern_tma_kernel<T, D, G>, smem) != cudaSuccess) return SANTA_ERR_CUDA;
      if (launch(bern_tma_kernel<T, D, G>, dim3(grid), dim3(32 * (kBtWarps + kBtProducers)), smem, a.st, true, p, items) !=
          cudaSuccess)
        return SANTA_ERR_CUDA;
      return SANTA_OK;
    }
  }
  if constexpr (sizeof(T) == 2) {
    if (for_decode && p.sub64) {  // decode on 64-key chunks: the persistent stream (bern_stream_kernel)
      const int nblk = (a.g->max_seqlen + kBernBlockKeys - 1) / kBernBlockKeys;
      const int items = a.g->batch * a.g->n_kv_heads * nblk;
      const int grid = std::min(items, 2 * num_sms());
      if (launch(bern_stream_kernel<T, D, G>, dim3(grid), dim3(32 * kBernStreamWarps), 0, a.st, true, p, items) !=
          cudaSuccess)
        return SANTA_ERR_CUDA;
      return SANTA_OK;
    }
  }
  if (launch(bern_chunk_kernel<T, D, G>, dim3(a.L.Cmax256, a.g->n_kv_heads, a.g->batch), dim3(kScoreThreads), 0,
             a.st, true, p) != cudaSuccess)
    return SANTA_ERR_CUDA;
  return SANTA_OK;
}

}  // namespace santa_host
