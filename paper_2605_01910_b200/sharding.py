"""Multi-GPU orchestration of the SANTA decode step (one process per GPU,
torch.distributed for the plumbing).

1. Batch x kv-head sharding (configs 2/3): the B*H_kv (batch, kv-head) units are independent,
   so they are partitioned into contiguous slabs, one or more per rank, with NO collective on
   the data path.  Philox is keyed by GLOBAL (b, h) through the geometry's batch_offset /
   head_offset, so every rank reproduces exactly the indices a single GPU would draw.

2. Sequence sharding (config 4, reading #18 of DESIGN.md): rank r holds the contiguous token
   range [r*n/R, (r+1)*n/R) of every sequence.  Phase 1 (local score pass) gives per-(b, h)
   (m_r, L_r); one all_gather of those [B, H, 2] fp64 tuples lets every rank build the same
   global shard CDF; phase 2 keeps the strata whose global threshold lands in the rank's slice of
   the CDF and gathers its local V rows; one all_reduce(SUM) of the [B, H, d] fp32 partials gives
   the output.  The sampled indices equal the unsharded ones (up to boundary rounding).

The two collectives run either through torch.distributed (NCCL) or through ``PeerExchange``: one-shot
peer-memory kernels of libsanta (santa_peer_allgather / santa_peer_allreduce_f32) that store straight
into every peer's CUDA-IPC-mapped exchange buffer over NVLink and sum the partials in fixed rank order.

The per-rank compute is a pluggable backend (``CudaBackend`` below = the C-ABI kernels); the
functions here only move tensors between ranks.  CPU tests drive the same orchestration with
world_size 2 over gloo and an oracle backend supplied by the test.
"""
from __future__ import annotations

import dataclasses
from typing import List, Optional, Tuple

import torch
import torch.distributed as dist


# ---------------------------------------------------------------------------------------------
# 1. batch x kv-head sharding
# ---------------------------------------------------------------------------------------------

@dataclasses.dataclass(frozen=True)
class Slab:
    """A rectangle of (batch, kv-head) units: batches [b0, b1) x kv-heads [k0, k1)."""
    b0: int
    b1: int
    k0: int
    k1: int

    @property
    def units(self) -> int:
        return (self.b1 - self.b0) * (self.k1 - self.k0)


def plan_units(batch: int, n_kv_heads: int, world: int) -> List[List[Slab]]:
    """Split the batch*n_kv_heads units (row-major over (b, kv-head)) into `world` contiguous
    ranges of near-equal size; each range is returned as at most three rectangular slabs
    (partial first batch, whole middle batches, partial last batch)."""
    if world < 1:
        raise ValueError("world must be >= 1")
    total = batch * n_kv_heads
    plan = []
    for r in range(world):
        u0, u1 = total * r // world, total * (r + 1) // world
        slabs = []
        u = u0
        while u < u1:
            b, k = divmod(u, n_kv_heads)
            if k == 0 and u1 - u >= n_kv_heads:   # whole batches
                nb = (u1 - u) // n_kv_heads
                slabs.append(Slab(b, b + nb, 0, n_kv_heads))
                u += nb * n_kv_heads
            else:                                  # part of one batch
                k1 = min(n_kv_heads, k + (u1 - u))
                slabs.append(Slab(b, b + 1, k, k1))
                u += k1 - k
        plan.append(slabs)
    return plan


def slab_inputs(q: torch.Tensor, K: torch.Tensor, V: torch.Tensor, seqlens: torch.Tensor, slab: Slab, G: int):
    """Views of a contiguous [B, H_kv, n, d] cache (and q [B, H, d]) restricted to one slab,
    made contiguous for the call (on a real deployment each rank only ever holds its slab)."""
    qs = q[slab.b0:slab.b1, slab.k0 * G:slab.k1 * G].contiguous()
    Ks = K[slab.b0:slab.b1, slab.k0:slab.k1].contiguous()
    Vs = V[slab.b0:slab.b1, slab.k0:slab.k1].contiguous()
    return qs, Ks, Vs, seqlens[slab.b0:slab.b1].contiguous()


# ---------------------------------------------------------------------------------------------
# 2. sequence sharding
# ---------------------------------------------------------------------------------------------

def shard_bounds(n: int, world: int) -> List[Tuple[int, int]]:
    """Contiguous shards in rank order: rank r holds tokens [r*n//R, (r+1)*n//R)."""
    return [(r * n // world, (r + 1) * n // world) for r in range(world)]


class CudaBackend:
    """Per-rank compute through the C-ABI (santa_seqshard_stats / santa_seqshard_sample_gather)."""

    def __init__(self):
        from . import (make_geometry, santa_seqshard_sample_gather, santa_seqshard_stats,  # noqa: F401
                       workspace)
        self._mk, self._ws_fn = make_geometry, workspace
        self._stats, self._sg = santa_seqshard_stats, santa_seqshard_sample_gather
        self.ws = None

    def stats(self, q, K_shard, shard_seqlens, n_kv_heads: int, S: int):
        geo = self._mk(q, n_kv_heads, K_shard.shape[2])
        if self.ws is None or self.ws.numel() < self._ws_bytes(geo, S):
            self.ws = self._ws_fn(geo, S, q.device)
        out = torch.empty(q.shape[0], q.shape[1], 2, dtype=torch.float64, device=q.device)
        self._stats(geo, q, K_shard, shard_seqlens, out, self.ws)
        self._geo = geo
        return out

    def _ws_bytes(self, geo, S):
        from . import santa_workspace_bytes
        return santa_workspace_bytes(geo, S)

    def sample_gather(self, stats_all, rank, world, token_offset, V_shard, shard_seqlens, S, mode, seed, offset,
                      return_idx=False):
        B, H = stats_all.shape[1], stats_all.shape[2]
        d = V_shard.shape[-1]
        partial = torch.empty(B, H, d, dtype=torch.float32, device=V_shard.device)
        idx = torch.empty(B, H, S, dtype=torch.int32, device=V_shard.device) if return_idx else None
        self._sg(self._geo, stats_all.contiguous(), rank, world, token_offset, V_shard, shard_seqlens, S, mode, seed,
                 offset, partial, idx, self.ws)
        return partial, idx


def shard_ranges(seqlens, rank: int, world: int, device=None):
    """This rank's contiguous token range of every sequence: (token_offset [B] int32, shard_len [B]
    int32), rank r holding [r*n//R, (r+1)*n//R).  Host logic; computed once per sequence-length
    change (a decode loop reuses it across steps -- no device sync on the step path)."""
    lens = [int(s) for s in (seqlens.tolist() if torch.is_tensor(seqlens) else seqlens)]
    lo = torch.tensor([rank * s // world for s in lens], dtype=torch.int32)
    hi = torch.tensor([(rank + 1) * s // world for s in lens], dtype=torch.int32)
    return lo.to(device) if device is not None else lo, (hi - lo).to(device) if device is not None else hi - lo


class PeerExchange:
    """One-shot peer-memory collectives for one rank per process (n_local = 1): an exchange buffer
    per rank, exported with CUDA IPC and mapped into every other rank (handles swapped once with
    all_gather_object over the process group), then each collective is ONE libsanta kernel.
    ``epoch`` counts the calls; every rank must issue the same sequence of calls."""

    def __init__(self, max_payload_bytes: int, group=None, device=None):
        from . import make_peer_group, santa_ipc_export, santa_ipc_import, santa_peer_buffer_bytes
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.nbytes = santa_peer_buffer_bytes(self.world, max_payload_bytes)
        if self.nbytes == 0:
            raise ValueError("PeerExchange: world must be 1..8")
        self.max_payload = max_payload_bytes
        self.buf = torch.zeros(self.nbytes, dtype=torch.uint8, device=device)
        torch.cuda.synchronize(self.buf.device)
        # every rank takes part in every collective below whatever fails locally, and all ranks raise
        # together if any rank could not export / map (no rank is left waiting in a collective)
        err = None
        try:
            mine = santa_ipc_export(self.buf)
        except Exception as e:  # noqa: BLE001
            mine, err = None, e
        handles = [None] * self.world
        dist.all_gather_object(handles, mine, group=group)
        self._bases, ptrs = [], []
        if err is None and all(h is not None for h in handles):
            try:
                for r, (h, off) in enumerate(handles):
                    if r == self.rank:
                        ptrs.append(self.buf.data_ptr())
                    else:
                        p, base = santa_ipc_import(h, off)
                        ptrs.append(p)
                        self._bases.append(base)
            except Exception as e:  # noqa: BLE001
                err = e
        ok = torch.tensor([1.0 if err is None and len(ptrs) == self.world else 0.0], device=self.buf.device)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=group)
        if ok.item() != 1.0:
            from . import santa_ipc_close
            for b in self._bases:
                santa_ipc_close(b)
            self._bases = []
            raise RuntimeError(f"PeerExchange: exchange buffers could not be mapped on every rank ({err!r})")
        self.peer_group = make_peer_group(ptrs, self.nbytes)
        self.epoch = 0

    def all_gather(self, t: torch.Tensor) -> torch.Tensor:
        from . import santa_peer_allgather
        t = t.contiguous()
        out = torch.empty((self.world,) + tuple(t.shape), dtype=t.dtype, device=t.device)
        self.epoch += 1
        santa_peer_allgather(self.peer_group, [self.rank], [t], [out], self.epoch)
        return out

    def all_reduce_(self, t: torch.Tensor) -> torch.Tensor:
        from . import santa_peer_allreduce_f32
        self.epoch += 1
        santa_peer_allreduce_f32(self.peer_group, [self.rank], [t], [t], self.epoch)
        return t

    def close(self):
        from . import santa_ipc_close
        torch.cuda.synchronize(self.buf.device)
        dist.barrier(group=self.group)      # no peer still writes into a mapping we drop
        for b in self._bases:
            santa_ipc_close(b)
        self._bases = []


class EmulatedPeerGroup:
    """All ranks of a group on ONE GPU (tests and single-GPU timing): every rank's exchange buffer
    is a local allocation and each collective serves all ranks in one cooperative launch
    (n_local = world) -- the only supported way to run ranks that wait on each other on one GPU."""

    def __init__(self, world: int, max_payload_bytes: int, device="cuda"):
        from . import make_peer_group, santa_peer_buffer_bytes
        self.world = world
        self.nbytes = santa_peer_buffer_bytes(world, max_payload_bytes)
        if self.nbytes == 0:
            raise ValueError("EmulatedPeerGroup: world must be 1..8")
        self.bufs = [torch.zeros(self.nbytes, dtype=torch.uint8, device=device) for _ in range(world)]
        self.peer_group = make_peer_group([b.data_ptr() for b in self.bufs], self.nbytes)
        self.epoch = 0

    def all_gather(self, ts):
        from . import santa_peer_allgather
        ts = [t.contiguous() for t in ts]
        outs = [torch.empty((self.world,) + tuple(t.shape), dtype=t.dtype, device=t.device) for t in ts]
        self.epoch += 1
        santa_peer_allgather(self.peer_group, list(range(self.world)), ts, outs, self.epoch)
        return outs

    def all_reduce_(self, ts):
        from . import santa_peer_allreduce_f32
        self.epoch += 1
        santa_peer_allreduce_f32(self.peer_group, list(range(self.world)), ts, ts, self.epoch)
        return ts


def seqshard_decode(q: torch.Tensor, K_shard: torch.Tensor, V_shard: torch.Tensor, seqlens: torch.Tensor,
                    S: int, mode: str, seed: int, offset: int = 0, backend=None, group=None,
                    return_idx: bool = False, ranges=None, exchange: Optional[PeerExchange] = None):
    """Sequence-sharded S^2ANTA decode step (config 4).  Every rank passes its own contiguous
    K/V shard [B, H_kv, n_local, d] and the FULL q [B, H, d] and seqlens [B] (global lengths).
    ``ranges``: this rank's (token_offset, shard_len) from shard_ranges(), precomputed by a decode
    loop (else derived from seqlens here, with a device-to-host read).
    ``exchange``: a PeerExchange to run both collectives as one-shot peer-memory kernels (else
    torch.distributed: NCCL all_gather_into_tensor / all_reduce, gloo all_gather / all_reduce).
    Returns the summed output [B, H, d] fp32 on every rank (and this rank's global indices, -1
    for strata owned by other ranks, if return_idx)."""
    backend = backend or CudaBackend()
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    n_loc = K_shard.shape[2]
    if ranges is None:
        ranges = shard_ranges(seqlens, rank, world, q.device)
        if int(ranges[1].max()) > n_loc:
            raise ValueError("K_shard too short for this rank's token range")
    lo, shard_len = ranges
    stats = backend.stats(q, K_shard, shard_len, K_shard.shape[1], S)           # [B, H, 2] fp64
    if exchange is not None:
        stats_all = exchange.all_gather(stats)                                  # one-shot P2P kernel
        partial, idx = backend.sample_gather(stats_all, rank, world, lo, V_shard, shard_len, S, mode, seed,
                                             offset, return_idx=return_idx)
        exchange.all_reduce_(partial)                                           # fixed rank order
        return (partial, idx) if return_idx else partial
    stats_all = torch.empty((world,) + tuple(stats.shape), dtype=stats.dtype, device=stats.device)
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(stats_all, stats, group=group)              # the exchange step
    else:
        dist.all_gather(list(stats_all.unbind(0)), stats, group=group)
    # stats_all: [R, B, H, 2]
    partial, idx = backend.sample_gather(stats_all, rank, world, lo, V_shard, shard_len, S, mode, seed,
                                         offset, return_idx=return_idx)
    dist.all_reduce(partial, op=dist.ReduceOp.SUM, group=group)                 # sum of partial outputs
    return (partial, idx) if return_idx else partial


def batch_shard_decode(q, K, V, seqlens, S, mode, seed, offset=0, group=None, decode_fn=None):
    """Batch x kv-head sharded decode: this rank computes its slabs of the (b, kv-head) units with
    global Philox ids; no collective.  Returns [(slab, out_slab)] for this rank."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    G = q.shape[1] // K.shape[1]
    if decode_fn is None:
        from . import decode as decode_fn  # noqa: N813
    res = []
    for slab in plan_units(q.shape[0], K.shape[1], world)[rank]:
        qs, Ks, Vs, sl = slab_inputs(q, K, V, seqlens, slab, G)
        out = decode_fn(qs, Ks, Vs, sl, S, mode, seed, offset, batch_offset=slab.b0, head_offset=slab.k0 * G)
        res.append((slab, out))
    return res
