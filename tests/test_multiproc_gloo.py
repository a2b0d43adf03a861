"""World-size-2 gloo tests of the multi-GPU orchestration (-m "not gpu").  The per-rank compute
is an oracle backend supplied HERE (the product package never imports the oracle); the test
checks that the sharded protocols (batch x kv-head slabs; sequence shards with the (m_r, L_r)
all-gather and the partial-output all-reduce) reproduce the unsharded oracle exactly."""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import santa_oracle as o
from paper_2605_01910_b200 import sharding

import santa_inputs as si


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class OracleBackend:
    """Per-rank compute of the sequence-sharded protocol with the fp64 oracle (test only)."""

    def __init__(self, G):
        self.G = G

    def stats(self, q, K_shard, shard_len, n_kv_heads, S):
        qf = o.to_f64(si.as_bits(q))
        Kf = o.to_f64(si.as_bits(K_shard))
        B, H, d = qf.shape
        self.s_local = {}
        out = torch.zeros(B, H, 2, dtype=torch.float64)
        for b in range(B):
            n = int(shard_len[b])
            for h in range(H):
                s = o.scores(qf[b, h], Kf[b, h // self.G, :n], 1 / math.sqrt(d))
                self.s_local[(b, h)] = s
                m, L = o.shard_stats(s)
                out[b, h, 0], out[b, h, 1] = m, L
        return out

    def sample_gather(self, stats_all, rank, world, token_offset, V_shard, shard_len, S, mode, seed, offset,
                      return_idx=False):
        Vf = o.to_f64(si.as_bits(V_shard))
        R, B, H, _ = stats_all.shape
        d = Vf.shape[-1]
        partial = torch.zeros(B, H, d, dtype=torch.float32)
        idx = torch.full((B, H, S), -1, dtype=torch.int32)
        for b in range(B):
            for h in range(H):
                st = [(float(stats_all[r, b, h, 0]), float(stats_all[r, b, h, 1])) for r in range(R)]
                T = o.thresholds(mode, S, o.sampler_uniforms(mode, S, seed, offset, h, b))
                mine, ids = o.shard_sample(self.s_local[(b, h)], int(token_offset[b]), st, rank, T)
                acc = np.zeros(d)
                for j in ids - int(token_offset[b]):
                    acc += Vf[b, h // self.G, j]
                partial[b, h] = torch.from_numpy(acc / S)
                idx[b, h, mine] = torch.from_numpy(ids.astype(np.int32))
        return partial, idx


def _seqshard_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        B, H, Hkv, d, n, S = 2, 8, 2, 32, [300, 157], 64
        inp = si.make_decode_inputs(B, H, Hkv, d, n, dtype="bf16", seed=21, workload="temp4")
        bounds = [sharding.shard_bounds(x, world)[rank] for x in n]
        nloc = max(b - a for a, b in bounds)
        Ks = torch.zeros(B, Hkv, nloc, d, dtype=inp.K.dtype)
        Vs = torch.zeros_like(Ks)
        for b, (a, e) in enumerate(bounds):
            Ks[b, :, :e - a] = inp.K[b, :, a:e]
            Vs[b, :, :e - a] = inp.V[b, :, a:e]
        out, idx = sharding.seqshard_decode(inp.q, Ks, Vs, inp.seqlens, S, "stratified", seed=7, offset=2,
                                            backend=OracleBackend(H // Hkv), return_idx=True)
        gathered = [torch.empty_like(idx) for _ in range(world)]
        dist.all_gather(gathered, idx)
        if rank == 0:
            out_ref, idx_ref = o.santa_decode(si.as_bits(inp.q), si.as_bits(inp.K), si.as_bits(inp.V), n, S,
                                              "stratified", 7, 2)
            own = torch.stack(gathered)                       # [R, B, H, S], -1 where not owned
            assert torch.all((own >= 0).sum(0) == 1), "every stratum owned by exactly one rank"
            merged = own.max(0).values.numpy()
            assert np.array_equal(merged, idx_ref)
            np.testing.assert_allclose(out.numpy(), out_ref, atol=1e-5)
            q.put("ok")
    except Exception as e:  # surface worker failures to the parent
        q.put(repr(e))
        raise
    finally:
        dist.destroy_process_group()


def _batchshard_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        B, H, Hkv, d, n, S = 3, 8, 4, 32, [40, 90, 17], 16
        G = H // Hkv
        inp = si.make_decode_inputs(B, H, Hkv, d, n, dtype="bf16", seed=22)

        def oracle_decode(qs, Ks, Vs, sl, S_, mode, seed, offset, batch_offset, head_offset):
            out, _ = o.santa_decode(si.as_bits(qs), si.as_bits(Ks), si.as_bits(Vs), sl.tolist(), S_, mode, seed,
                                    offset, batch_offset=batch_offset, head_offset=head_offset)
            return torch.from_numpy(out)

        mine = sharding.batch_shard_decode(inp.q, inp.K, inp.V, inp.seqlens, S, "systematic", 5, 0,
                                           decode_fn=oracle_decode)
        full = torch.zeros(B, H, d, dtype=torch.float64)
        for slab, out in mine:
            full[slab.b0:slab.b1, slab.k0 * G:slab.k1 * G] = out
        dist.all_reduce(full)
        if rank == 0:
            ref, _ = o.santa_decode(si.as_bits(inp.q), si.as_bits(inp.K), si.as_bits(inp.V), n, S, "systematic", 5)
            np.testing.assert_array_equal(full.numpy(), ref)
            q.put("ok")
    except Exception as e:
        q.put(repr(e))
        raise
    finally:
        dist.destroy_process_group()


def _run(worker, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    mp.start_processes(worker, args=(world, _free_port(), q), nprocs=world, join=True, start_method="spawn")
    assert q.get(timeout=5) == "ok"


def test_plan_units_partitions_every_unit_once():
    for B, Hkv, world in [(1, 8, 8), (32, 8, 8), (3, 8, 2), (5, 3, 4), (2, 8, 3), (1, 1, 1)]:
        seen = []
        plan = sharding.plan_units(B, Hkv, world)
        assert len(plan) == world
        for slabs in plan:
            for s in slabs:
                assert 0 <= s.b0 < s.b1 <= B and 0 <= s.k0 < s.k1 <= Hkv
                seen += [(b, k) for b in range(s.b0, s.b1) for k in range(s.k0, s.k1)]
        assert sorted(seen) == [(b, k) for b in range(B) for k in range(Hkv)]
        sizes = [sum(s.units for s in slabs) for slabs in plan]
        assert max(sizes) - min(sizes) <= 1


def test_sequence_sharded_protocol_gloo_world2():
    _run(_seqshard_worker)


def test_batch_kvhead_sharding_gloo_world2():
    _run(_batchshard_worker)
