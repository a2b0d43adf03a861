"""paper_2605_01910_b200 -- B200-native SANTA / S^2ANTA stochastic sparse decode attention
(arXiv 2605.01910).

Thin Python binding over the C-ABI library ``libsanta.so`` (include/santa.h): the
functions below have the ABI's names and only marshal torch tensors into pointers; every
step of the hot path (scores, softmax statistics, CDF, Philox thresholds, inverse CDF,
gather-add) runs in the sm_100a CUDA kernels.  There is no CPU fallback: importing this
package without the built library raises ImportError, and calling it on CPU tensors
raises ValueError.
"""
from __future__ import annotations

import ctypes
from typing import Optional, Sequence

import torch

from . import _abi
from ._abi import (DTYPES, FLAG_EMPTY_SEQ, FLAG_PEER_TIMEOUT, FLAG_SYNC_TIMEOUT, MODES, PATHS, Geometry,
                   LayerSchedule, PeerGroup, SantaError)

__all__ = [
    "Geometry", "SantaError", "MODES", "make_geometry", "workspace", "santa_workspace_bytes", "santa_auto_path",
    "santa_decode_attention", "santa_decode_attention_path", "santa_decode_attention_profiled", "santa_score_phase",
    "santa_sample_phase", "PATHS", "FLAG_SYNC_TIMEOUT",
    "santa_dense_reference", "santa_decode_attention_prop", "santa_prop_tile_len", "santa_decode_attention_flash",
    "santa_flash_max_samples", "decode_flash",
    "santa_bernoulli_scores", "santa_decode_attention_bernoulli", "santa_seqshard_stats",
    "santa_seqshard_sample_gather", "santa_decode_step_host", "santa_decode_step_host_packed", "santa_philox_uniforms",
    "santa_read_error_flags", "santa_version", "decode", "decode_prop", "dense", "LIB_PATH",
    "santa_decode_attention_append", "LayerSchedule", "make_schedule", "santa_schedule_workspace_bytes",
    "santa_decode_attention_layer", "decode_append", "prepare_decode",
    "PeerGroup", "FLAG_PEER_TIMEOUT", "make_peer_group", "santa_peer_buffer_bytes", "santa_peer_allgather",
    "santa_peer_allreduce_f32", "santa_ipc_export", "santa_ipc_import", "santa_ipc_close",
]
LIB_PATH = _abi.LIB_PATH
_TORCH_DT = {torch.bfloat16: "bf16", torch.float32: "f32", torch.float16: "f16"}


def _ptr(t: Optional[torch.Tensor]):
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("libsanta takes CUDA tensors only (no CPU path)")
    if not t.is_contiguous():
        raise ValueError("tensors must be contiguous")
    return ctypes.c_void_p(t.data_ptr())


def _stream(stream) -> ctypes.c_void_p:
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))


def make_geometry(q: torch.Tensor, n_kv_heads: int, max_seqlen: int, page_table: Optional[torch.Tensor] = None,
                  page_size: int = 0, scale: float = 0.0, batch_offset: int = 0, head_offset: int = 0) -> Geometry:
    """Geometry struct for q [B, H, d] and a cache with n_kv_heads heads (see santa.h)."""
    B, H, d = q.shape
    g = Geometry()
    g.batch, g.n_heads, g.n_kv_heads, g.head_dim = B, H, n_kv_heads, d
    g.dtype = DTYPES[_TORCH_DT[q.dtype]]
    g.page_table = page_table.data_ptr() if page_table is not None else None
    g.page_size = page_size if page_table is not None else 0
    g.max_pages_per_seq = page_table.shape[1] if page_table is not None else 0
    g.max_seqlen = max_seqlen
    g.scale = scale
    g.batch_offset, g.head_offset = batch_offset, head_offset
    return g


def santa_version() -> str:
    return _abi.LIB.santa_version().decode()


def santa_workspace_bytes(geo: Geometry, S: int) -> int:
    return int(_abi.LIB.santa_workspace_bytes(ctypes.byref(geo), S))


def santa_auto_path(geo: Geometry, S: int) -> str:
    """The execution path santa_decode_attention takes ("two_kernel", "step" or "step_tc")."""
    code = int(_abi.LIB.santa_auto_path(ctypes.byref(geo), S))
    if code < 0:
        raise SantaError("santa_auto_path", 1)
    return {v: k for k, v in PATHS.items()}[code]


def workspace(geo: Geometry, S: int, device="cuda") -> torch.Tensor:
    n = santa_workspace_bytes(geo, S)
    if n == 0:
        raise SantaError("santa_workspace_bytes", 1)
    # zero-initialised: the single-launch step kernel keeps its self-cleaning sync counters here
    return torch.zeros(n, dtype=torch.uint8, device=device)


def santa_decode_attention(geo, q, K, V, seqlens, S, mode, seed, offset, out, idx_out, ws, stream=None):
    _abi.check("santa_decode_attention", _abi.LIB.santa_decode_attention(
        ctypes.byref(geo), _ptr(q), _ptr(K), _ptr(V), _ptr(seqlens), S, MODES.get(mode, mode), seed, offset,
        _ptr(out), _ptr(idx_out), _ptr(ws), ws.numel(), _stream(stream)))


def prepare_decode(geo, q, K, V, seqlens, S, mode, seed, out, idx_out, ws, path="auto", stream=None):
    """A decode step with every argument but the Philox offset marshalled once: returns launch(offset),
    which issues santa_decode_attention_path on the prepared buffers (the per-step host cost of a
    decode loop drops to one ctypes call).  The tensors must stay alive and in place."""
    fn = _abi.LIB.santa_decode_attention_path
    args = (ctypes.byref(geo), _ptr(q), _ptr(K), _ptr(V), _ptr(seqlens), ctypes.c_int32(S),
            ctypes.c_int32(MODES.get(mode, mode)), ctypes.c_uint64(seed))
    tail = (_ptr(out), _ptr(idx_out), _ptr(ws), ctypes.c_size_t(ws.numel()), ctypes.c_int32(PATHS.get(path, path)),
            _stream(stream))
    keep = (geo, q, K, V, seqlens, out, idx_out, ws)

    def launch(offset: int):
        st = fn(*args, ctypes.c_uint64(offset), *tail)
        if st != 0:
            _abi.check("santa_decode_attention_path", st)
    launch._keep = keep
    return launch


def santa_decode_attention_path(geo, q, K, V, seqlens, S, mode, seed, offset, out, idx_out, ws, path,
                                stream=None):
    """path: "auto" | "step" (single pipelined launch) | "two_kernel" (score pass + sampler)."""
    _abi.check("santa_decode_attention_path", _abi.LIB.santa_decode_attention_path(
        ctypes.byref(geo), _ptr(q), _ptr(K), _ptr(V), _ptr(seqlens), S, MODES.get(mode, mode), seed, offset,
        _ptr(out), _ptr(idx_out), _ptr(ws), ws.numel(), PATHS.get(path, path), _stream(stream)))


def santa_decode_attention_profiled(geo, q, K, V, seqlens, S, mode, seed, offset, out, idx_out, ws, events,
                                    stream=None):
    ev = (ctypes.c_void_p * 3)(*[ctypes.c_void_p(e.cuda_event) for e in events])
    _abi.check("santa_decode_attention_profiled", _abi.LIB.santa_decode_attention_profiled(
        ctypes.byref(geo), _ptr(q), _ptr(K), _ptr(V), _ptr(seqlens), S, MODES.get(mode, mode), seed, offset,
        _ptr(out), _ptr(idx_out), _ptr(ws), ws.numel(), ctypes.cast(ev, ctypes.c_void_p), _stream(stream)))


def santa_score_phase(geo, q, K, seqlens, ws, stream=None):
    _abi.check("santa_score_phase", _abi.LIB.santa_score_phase(
        ctypes.byref(geo), _ptr(q), _ptr(K), _ptr(seqlens), _ptr(ws), ws.numel(), _stream(stream)))


def santa_sample_phase(geo, V, seqlens, S, mode, seed, offset, out, idx_out, ws, stream=None):
    _abi.check("santa_sample_phase", _abi.LIB.santa_sample_phase(
        ctypes.byref(geo), _ptr(V), _ptr(seqlens), S, MODES.get(mode, mode), seed, offset, _ptr(out), _ptr(idx_out),
        _ptr(ws), ws.numel(), _stream(stream)))


def santa_decode_attention_prop(geo, q, K, V, seqlens, S, seed, offset, out, idx_out, ws, stream=None):
    """S^2ANTA-prop (largest-remainder tile budgets, per-tile systematic counts; include/santa.h)."""
    _abi.check("santa_decode_attention_prop", _abi.LIB.santa_decode_attention_prop(
        ctypes.byref(geo), _ptr(q), _ptr(K), _ptr(V), _ptr(seqlens), S, seed, offset, _ptr(out), _ptr(idx_out),
        _ptr(ws), ws.numel(), _stream(stream)))


def santa_prop_tile_len(geo: Geometry) -> int:
    """B_tile of santa_decode_attention_prop for this geometry (pure host logic)."""
    n = int(_abi.LIB.santa_prop_tile_len(ctypes.byref(geo)))
    if n < 1:
        raise SantaError("santa_prop_tile_len", 1)
    return n


def santa_decode_attention_flash(geo, q, K, V, seqlens, S, tile_len, seed, offset, out, idx_out, ws, stream=None):
    """S^2ANTA-flash (uniform per-tile budgets + LSE merge; include/santa.h)."""
    _abi.check("santa_decode_attention_flash", _abi.LIB.santa_decode_attention_flash(
        ctypes.byref(geo), _ptr(q), _ptr(K), _ptr(V), _ptr(seqlens), S, tile_len, seed, offset, _ptr(out),
        _ptr(idx_out), _ptr(ws), ws.numel(), _stream(stream)))


def santa_flash_max_samples(geo: Geometry, S: int, tile_len: int) -> int:
    """idx_out row length of santa_decode_attention_flash (pure host logic)."""
    n = int(_abi.LIB.santa_flash_max_samples(ctypes.byref(geo), S, tile_len))
    if n < 1:
        raise SantaError("santa_flash_max_samples", 1)
    return n


def santa_dense_reference(geo, q, K, V, seqlens, out, ws, stream=None):
    _abi.check("santa_dense_reference", _abi.LIB.santa_dense_reference(
        ctypes.byref(geo), _ptr(q), _ptr(K), _ptr(V), _ptr(seqlens), _ptr(out), _ptr(ws), ws.numel(),
        _stream(stream)))


def santa_bernoulli_scores(geo, q, Kt, seqlens, B, stratified, mean_group, seed, offset, scores, feature_mask, ws,
                           stream=None):
    _abi.check("santa_bernoulli_scores", _abi.LIB.santa_bernoulli_scores(
        ctypes.byref(geo), _ptr(q), _ptr(Kt), _ptr(seqlens), B, int(stratified), int(mean_group), seed, offset,
        _ptr(scores), _ptr(feature_mask), _ptr(ws), ws.numel(), _stream(stream)))


def santa_decode_attention_bernoulli(geo, q, Kt, V, seqlens, B, stratified, mean_group, S, mode, seed, offset, out,
                                     idx_out, ws, stream=None):
    _abi.check("santa_decode_attention_bernoulli", _abi.LIB.santa_decode_attention_bernoulli(
        ctypes.byref(geo), _ptr(q), _ptr(Kt), _ptr(V), _ptr(seqlens), B, int(stratified), int(mean_group), S,
        MODES.get(mode, mode), seed, offset, _ptr(out), _ptr(idx_out), _ptr(ws), ws.numel(), _stream(stream)))


def santa_seqshard_stats(geo, q, K_shard, shard_seqlens, stats_out, ws, stream=None):
    _abi.check("santa_seqshard_stats", _abi.LIB.santa_seqshard_stats(
        ctypes.byref(geo), _ptr(q), _ptr(K_shard), _ptr(shard_seqlens), _ptr(stats_out), _ptr(ws), ws.numel(),
        _stream(stream)))


def santa_seqshard_sample_gather(geo, stats_all, rank, world, token_offset, V_shard, shard_seqlens, S, mode, seed,
                                 offset, partial_out, idx_out, ws, stream=None):
    _abi.check("santa_seqshard_sample_gather", _abi.LIB.santa_seqshard_sample_gather(
        ctypes.byref(geo), _ptr(stats_all), rank, world, _ptr(token_offset), _ptr(V_shard), _ptr(shard_seqlens), S,
        MODES.get(mode, mode), seed, offset, _ptr(partial_out), _ptr(idx_out), _ptr(ws), ws.numel(),
        _stream(stream)))


def santa_decode_step_host(geo, q_host, k_new_host, v_new_host, q_dev, k_new_dev, v_new_dev, K, V, seqlens, S, mode,
                           seed, offset, out_dev, out_host, ws, stream=None):
    for t in (q_host, k_new_host, v_new_host, out_host):
        if t.is_cuda or not t.is_pinned():
            raise ValueError("host buffers must be pinned CPU tensors")
    hp = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
    _abi.check("santa_decode_step_host", _abi.LIB.santa_decode_step_host(
        ctypes.byref(geo), hp(q_host), hp(k_new_host), hp(v_new_host), _ptr(q_dev), _ptr(k_new_dev),
        _ptr(v_new_dev), _ptr(K), _ptr(V), _ptr(seqlens), S, MODES.get(mode, mode), seed, offset, _ptr(out_dev),
        hp(out_host), _ptr(ws), ws.numel(), _stream(stream)))


def santa_decode_step_host_packed(geo, qkv_host, qkv_dev, K, V, seqlens, S, mode, seed, offset, out_dev, out_host,
                                  ws, synchronize=True, stream=None):
    """Packed [q | k_new | v_new] host buffer -> KV append + decode -> out host buffer.  Pinned buffers
    are read / written by the kernels (zero copy); pageable ones are copied (include/santa.h)."""
    for t in (qkv_host, out_host):
        if t.is_cuda or not t.is_contiguous():
            raise ValueError("host buffers must be contiguous CPU tensors")
    hp = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
    _abi.check("santa_decode_step_host_packed", _abi.LIB.santa_decode_step_host_packed(
        ctypes.byref(geo), hp(qkv_host), _ptr(qkv_dev), _ptr(K), _ptr(V), _ptr(seqlens), S, MODES.get(mode, mode),
        seed, offset, _ptr(out_dev), hp(out_host), _ptr(ws), ws.numel(), int(bool(synchronize)), _stream(stream)))


def santa_decode_attention_append(geo, q, K, V, k_new, v_new, seqlens, S, mode, seed, offset, out, idx_out, ws,
                                  stream=None):
    """Decode step with the current token's KV append (k_new / v_new [B, H_kv, d] written at slot
    seqlens[b] - 1 of K / V; fused into the score pass on the two-kernel path; include/santa.h)."""
    _abi.check("santa_decode_attention_append", _abi.LIB.santa_decode_attention_append(
        ctypes.byref(geo), _ptr(q), _ptr(K), _ptr(V), _ptr(k_new), _ptr(v_new), _ptr(seqlens), S,
        MODES.get(mode, mode), seed, offset, _ptr(out), _ptr(idx_out), _ptr(ws), ws.numel(), _stream(stream)))


def make_schedule(S_per_layer: Sequence[int]) -> LayerSchedule:
    """Per-layer sample budgets (App. K): a santa_layer_schedule over a host int32 array.  The array
    is kept alive on the returned struct."""
    arr = (ctypes.c_int32 * len(S_per_layer))(*[int(x) for x in S_per_layer])
    sched = LayerSchedule(len(S_per_layer), ctypes.cast(arr, ctypes.POINTER(ctypes.c_int32)))
    sched._keep = arr
    return sched


def santa_schedule_workspace_bytes(geo: Geometry, sched: LayerSchedule) -> int:
    return int(_abi.LIB.santa_schedule_workspace_bytes(ctypes.byref(geo), ctypes.byref(sched)))


def santa_decode_attention_layer(geo, sched, layer, q, K, V, k_new, v_new, seqlens, mode, seed, offset, out,
                                 idx_out, ws, stream=None):
    """Layer `layer` of a per-layer schedule: S = sched.S[layer], Philox offset offset*n_layers+layer;
    k_new / v_new None (no append) or the new token's rows."""
    _abi.check("santa_decode_attention_layer", _abi.LIB.santa_decode_attention_layer(
        ctypes.byref(geo), ctypes.byref(sched), layer, _ptr(q), _ptr(K), _ptr(V), _ptr(k_new), _ptr(v_new),
        _ptr(seqlens), MODES.get(mode, mode), seed, offset, _ptr(out), _ptr(idx_out), _ptr(ws), ws.numel(),
        _stream(stream)))


def santa_philox_uniforms(seed, offset, tag, h_global, b_global, n, out, ctr_key: Optional[Sequence[int]] = None,
                          raw_out=None, stream=None):
    ck = (ctypes.c_uint32 * 6)(*ctr_key) if ctr_key is not None else None
    _abi.check("santa_philox_uniforms", _abi.LIB.santa_philox_uniforms(
        seed, offset, tag, h_global, b_global, n, _ptr(out), ctypes.cast(ck, ctypes.c_void_p) if ck else None,
        _ptr(raw_out), _stream(stream)))


def santa_read_error_flags(ws, stream=None) -> int:
    f = ctypes.c_uint32(0)
    _abi.check("santa_read_error_flags", _abi.LIB.santa_read_error_flags(_ptr(ws), ctypes.byref(f), _stream(stream)))
    return int(f.value)


def santa_peer_buffer_bytes(world: int, max_payload_bytes: int) -> int:
    return int(_abi.LIB.santa_peer_buffer_bytes(world, max_payload_bytes))


def make_peer_group(bufs: Sequence[int], buf_bytes: int) -> PeerGroup:
    """santa_peer_group from every rank's buffer address (ints, as mapped into this process)."""
    g = PeerGroup()
    g.world = len(bufs)
    for r, p in enumerate(bufs):
        g.bufs[r] = int(p)
    g.buf_bytes = int(buf_bytes)
    return g


def _ptr_array(ptrs, ctype=ctypes.c_void_p):
    return (ctype * len(ptrs))(*ptrs)


def santa_peer_allgather(group: PeerGroup, ranks: Sequence[int], src: Sequence[torch.Tensor],
                         dst: Sequence[torch.Tensor], epoch: int, stream=None):
    """One-shot all-gather: src[l] (this call's rank ranks[l]) -> dst[l] = [world, *src shape]."""
    nbytes = src[0].numel() * src[0].element_size()
    for s_, d_ in zip(src, dst):
        if s_.numel() * s_.element_size() != nbytes or d_.numel() * d_.element_size() != group.world * nbytes:
            raise ValueError("allgather: src / dst sizes")
    _abi.check("santa_peer_allgather", _abi.LIB.santa_peer_allgather(
        ctypes.byref(group), len(ranks), _ptr_array(ranks, ctypes.c_int32), _ptr_array([_ptr(t) for t in src]),
        _ptr_array([_ptr(t) for t in dst]), nbytes, epoch, _stream(stream)))


def santa_peer_allreduce_f32(group: PeerGroup, ranks: Sequence[int], src: Sequence[torch.Tensor],
                             dst: Sequence[torch.Tensor], epoch: int, stream=None):
    """One-shot SUM in rank order: dst[l] = sum_r src of rank r (fp32; dst may be src)."""
    n = src[0].numel()
    for s_, d_ in zip(src, dst):
        if s_.dtype != torch.float32 or d_.dtype != torch.float32 or s_.numel() != n or d_.numel() != n:
            raise ValueError("allreduce_f32: fp32 tensors of equal size")
    _abi.check("santa_peer_allreduce_f32", _abi.LIB.santa_peer_allreduce_f32(
        ctypes.byref(group), len(ranks), _ptr_array(ranks, ctypes.c_int32), _ptr_array([_ptr(t) for t in src]),
        _ptr_array([_ptr(t) for t in dst]), n, epoch, _stream(stream)))


def santa_ipc_export(t: torch.Tensor):
    """(64-byte handle, offset) of a device tensor's allocation for santa_ipc_import elsewhere."""
    h = ctypes.create_string_buffer(_abi.IPC_HANDLE_BYTES)
    off = ctypes.c_size_t(0)
    _abi.check("santa_ipc_export", _abi.LIB.santa_ipc_export(_ptr(t), h, ctypes.byref(off)))
    return bytes(h.raw), int(off.value)


def santa_ipc_import(handle: bytes, offset: int):
    """Maps a peer's exported allocation: (device address of the peer tensor, mapping base)."""
    p, base = ctypes.c_void_p(), ctypes.c_void_p()
    hb = ctypes.create_string_buffer(bytes(handle), _abi.IPC_HANDLE_BYTES)
    _abi.check("santa_ipc_import", _abi.LIB.santa_ipc_import(hb, offset, ctypes.byref(p), ctypes.byref(base)))
    return int(p.value), int(base.value)


def santa_ipc_close(base: int):
    _abi.check("santa_ipc_close", _abi.LIB.santa_ipc_close(ctypes.c_void_p(base)))


# ---- convenience wrappers (allocation + the call; still no compute in Python) ----------------

def _check_cache(q, K, V, Hkv, n_max, page_table, page_size):
    """Shape/dtype agreement between q and the cache the geometry will describe.  For a contiguous
    cache the row stride of K and V IS max_seqlen (santa.h), so a max_seqlen different from
    K.shape[2] would silently read the wrong rows: refuse it."""
    if q.dim() != 3:
        raise ValueError(f"q must be [B, H, d], got {tuple(q.shape)}")
    B, H, d = q.shape
    if K.dtype != q.dtype or V.dtype != q.dtype:
        raise ValueError(f"q, K, V must share a dtype (got {q.dtype}, {K.dtype}, {V.dtype})")
    if K.shape != V.shape:
        raise ValueError(f"K and V shapes differ: {tuple(K.shape)} vs {tuple(V.shape)}")
    if page_table is None:
        if tuple(K.shape) != (B, Hkv, n_max, d):
            raise ValueError(f"contiguous cache must be [B, H_kv, max_seqlen, d] = {(B, Hkv, n_max, d)}, "
                             f"got {tuple(K.shape)}")
    else:
        if K.dim() != 4 or K.shape[1] != Hkv or K.shape[2] != page_size or K.shape[3] != d:
            raise ValueError(f"paged pool must be [pages, H_kv, page_size, d] = [*, {Hkv}, {page_size}, {d}], "
                             f"got {tuple(K.shape)}")
        if page_table.dtype != torch.int32 or page_table.dim() != 2 or page_table.shape[0] != B:
            raise ValueError("page_table must be int32 [B, max_pages_per_seq]")

def decode(q, K, V, seqlens, S, mode="stratified", seed=0, offset=0, n_kv_heads=None, page_table=None,
           page_size=0, max_seqlen=None, return_idx=False, ws=None, batch_offset=0, head_offset=0, path="auto"):
    """Allocate out (+ idx) and workspace, run santa_decode_attention.  K/V are either the
    contiguous [B, H_kv, n_max, d] cache or the paged pool [pages, H_kv, P, d]."""
    Hkv = n_kv_heads or K.shape[1]
    n_max = max_seqlen or (K.shape[2] if page_table is None else page_table.shape[1] * page_size)
    _check_cache(q, K, V, Hkv, n_max, page_table, page_size)
    geo = make_geometry(q, Hkv, n_max, page_table, page_size, batch_offset=batch_offset, head_offset=head_offset)
    if ws is None:
        ws = workspace(geo, S, q.device)
    out = torch.empty_like(q)
    idx = torch.empty((q.shape[0], q.shape[1], S), dtype=torch.int32, device=q.device) if return_idx else None
    santa_decode_attention_path(geo, q, K, V, seqlens, S, mode, seed, offset, out, idx, ws, path)
    return (out, idx) if return_idx else out


def decode_prop(q, K, V, seqlens, S, seed=0, offset=0, n_kv_heads=None, page_table=None, page_size=0,
                max_seqlen=None, return_idx=False, ws=None, batch_offset=0, head_offset=0):
    """Allocate out (+ idx) and workspace, run santa_decode_attention_prop (S^2ANTA-prop)."""
    Hkv = n_kv_heads or K.shape[1]
    n_max = max_seqlen or (K.shape[2] if page_table is None else page_table.shape[1] * page_size)
    _check_cache(q, K, V, Hkv, n_max, page_table, page_size)
    geo = make_geometry(q, Hkv, n_max, page_table, page_size, batch_offset=batch_offset, head_offset=head_offset)
    if ws is None:
        ws = workspace(geo, S, q.device)
    out = torch.empty_like(q)
    idx = torch.empty((q.shape[0], q.shape[1], S), dtype=torch.int32, device=q.device) if return_idx else None
    santa_decode_attention_prop(geo, q, K, V, seqlens, S, seed, offset, out, idx, ws)
    return (out, idx) if return_idx else out


def decode_flash(q, K, V, seqlens, S, tile_len=256, seed=0, offset=0, n_kv_heads=None, page_table=None,
                 page_size=0, max_seqlen=None, return_idx=False, ws=None, batch_offset=0, head_offset=0):
    """Allocate out (+ idx [B, H, santa_flash_max_samples]) and workspace, run santa_decode_attention_flash."""
    Hkv = n_kv_heads or K.shape[1]
    n_max = max_seqlen or (K.shape[2] if page_table is None else page_table.shape[1] * page_size)
    _check_cache(q, K, V, Hkv, n_max, page_table, page_size)
    geo = make_geometry(q, Hkv, n_max, page_table, page_size, batch_offset=batch_offset, head_offset=head_offset)
    if ws is None:
        ws = workspace(geo, S, q.device)
    out = torch.empty_like(q)
    idx = None
    if return_idx:
        M = santa_flash_max_samples(geo, S, tile_len)
        idx = torch.empty((q.shape[0], q.shape[1], M), dtype=torch.int32, device=q.device)
    santa_decode_attention_flash(geo, q, K, V, seqlens, S, tile_len, seed, offset, out, idx, ws)
    return (out, idx) if return_idx else out


def dense(q, K, V, seqlens, n_kv_heads=None, page_table=None, page_size=0, max_seqlen=None, ws=None):
    Hkv = n_kv_heads or K.shape[1]
    n_max = max_seqlen or (K.shape[2] if page_table is None else page_table.shape[1] * page_size)
    _check_cache(q, K, V, Hkv, n_max, page_table, page_size)
    geo = make_geometry(q, Hkv, n_max, page_table, page_size)
    if ws is None:
        ws = workspace(geo, 1, q.device)
    out = torch.empty_like(q)
    santa_dense_reference(geo, q, K, V, seqlens, out, ws)
    return out


def decode_append(q, K, V, k_new, v_new, seqlens, S, mode="stratified", seed=0, offset=0, return_idx=False, ws=None):
    """Allocate out (+ idx) and workspace, run santa_decode_attention_append on a contiguous cache."""
    Hkv = K.shape[1]
    _check_cache(q, K, V, Hkv, K.shape[2], None, 0)
    if k_new.shape != (q.shape[0], Hkv, q.shape[2]) or v_new.shape != k_new.shape or k_new.dtype != q.dtype:
        raise ValueError("k_new / v_new must be [B, H_kv, d] of the cache dtype")
    geo = make_geometry(q, Hkv, K.shape[2])
    if ws is None:
        ws = workspace(geo, S, q.device)
    out = torch.empty_like(q)
    idx = torch.empty((q.shape[0], q.shape[1], S), dtype=torch.int32, device=q.device) if return_idx else None
    santa_decode_attention_append(geo, q, K, V, k_new.contiguous(), v_new.contiguous(), seqlens, S, mode, seed,
                                  offset, out, idx, ws)
    return (out, idx) if return_idx else out
