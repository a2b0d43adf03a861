"""One-shot peer-memory collectives (santa_peer_allgather / santa_peer_allreduce_f32; config 4's
exchange) on one GPU (-m gpu).

One GPU cannot run ranks whose kernels wait on each other as separate launches, so every test
emulates the whole group in ONE cooperative launch (n_local = world; every rank's exchange buffer
is a local allocation) -- the same kernel, push / flag / wait / consume code a multi-GPU run
executes with n_local = 1.  Checks: the all-gather is a byte copy; the SUM equals the sequential
fp32 sum in rank order bit for bit (identical on every rank); buffer halves alternate safely over
many epochs; argument errors launch nothing; the config-4 step with the peer exchange equals the
by-hand exchange bit for bit and the unsharded run; the CUDA-IPC mapping works across processes."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2605_01910_b200 as santa
from paper_2605_01910_b200 import sharding
import santa_inputs as si
from test_gpu_fullsize import unit_parity

pytestmark = pytest.mark.gpu


def _payloads(world, nbytes, gen):
    return [torch.randint(-2**31, 2**31 - 1, (nbytes // 4,), dtype=torch.int32, generator=gen).cuda()
            for _ in range(world)]


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("nbytes", [16, 512, 16 * 37, 16384, 40000, 131072])
def test_allgather_emulated(world, nbytes):
    gen = torch.Generator().manual_seed(world * 1000 + nbytes)
    grp = sharding.EmulatedPeerGroup(world, 131072)
    for _ in range(3):   # both buffer halves, then the first again
        src = _payloads(world, nbytes, gen)
        outs = grp.all_gather(src)
        torch.cuda.synchronize()
        ref = torch.stack(src)
        for o in outs:
            assert torch.equal(o, ref)
    assert santa.santa_read_error_flags(grp.bufs[0]) == 0


@pytest.mark.parametrize("world", [1, 2, 3, 5, 8])
@pytest.mark.parametrize("n", [4, 4 * 33, 4096, 32 * 128, 64 * 32 * 128])
def test_allreduce_emulated_bit_exact(world, n):
    gen = torch.Generator().manual_seed(world * 7 + n)
    grp = sharding.EmulatedPeerGroup(world, n * 4)
    for it in range(3):
        src = [(torch.randn(n, generator=gen) * (10.0 ** (r % 3))).cuda() for r in range(world)]
        ref = src[0].clone()
        for r in range(1, world):
            ref = ref + src[r]            # sequential fp32 adds in rank order
        dst = [torch.empty_like(s) for s in src] if it % 2 else [s.clone() for s in src]
        if it % 2:
            santa.santa_peer_allreduce_f32(grp.peer_group, list(range(world)), src, dst, grp.epoch + 1)
            grp.epoch += 1
        else:
            grp.all_reduce_(dst)          # in place
        torch.cuda.synchronize()
        for d_ in dst:
            assert torch.equal(d_, ref)


def test_alternating_ops_many_epochs():
    """Gathers and reductions interleaved over 40 epochs on one group (both halves reused 20 times)."""
    world = 4
    grp = sharding.EmulatedPeerGroup(world, 16384)
    gen = torch.Generator().manual_seed(3)
    for e in range(40):
        if e % 3 == 0:
            src = [torch.randn(32 * 2, dtype=torch.float64, generator=gen).cuda() for _ in range(world)]
            outs = grp.all_gather(src)
            torch.cuda.synchronize()
            assert all(torch.equal(o, torch.stack(src)) for o in outs)
        else:
            src = [torch.randn(32 * 128, generator=gen).cuda() for _ in range(world)]
            ref = src[0] + src[1] + src[2] + src[3]
            grp.all_reduce_(src)
            torch.cuda.synchronize()
            assert all(torch.equal(s, ref) for s in src)


def test_argument_errors_launch_nothing():
    grp = sharding.EmulatedPeerGroup(2, 1024)
    src = [torch.ones(64, device="cuda") for _ in range(2)]
    dst = [torch.zeros(2 * 64, device="cuda") for _ in range(2)]
    with pytest.raises(santa.SantaError, match="INVALID_ARG"):
        santa.santa_peer_allgather(grp.peer_group, [0, 1], src, dst, 0)            # epoch 0
    with pytest.raises(santa.SantaError, match="INVALID_ARG"):
        santa.santa_peer_allgather(grp.peer_group, [1, 1], src, dst, 1)            # repeated rank
    big = [torch.ones(512, device="cuda") for _ in range(2)]
    with pytest.raises(santa.SantaError, match="WORKSPACE"):
        santa.santa_peer_allgather(grp.peer_group, [0, 1], big, [torch.zeros(1024, device="cuda")] * 2, 1)
    with pytest.raises(santa.SantaError, match="ALIGNMENT"):
        santa.santa_peer_allreduce_f32(grp.peer_group, [0, 1], [torch.ones(3, device="cuda")] * 2,
                                       [torch.ones(3, device="cuda")] * 2, 1)       # 12 B
    torch.cuda.synchronize()
    assert torch.all(dst[0] == 0) and torch.all(dst[1] == 0)
    assert int(grp.bufs[0].sum()) == 0 and int(grp.bufs[1].sum()) == 0


@pytest.mark.parametrize("R", [2, 4, 8])
def test_seqshard_step_with_peer_exchange(R):
    """Config 4's step (512k tokens, S = 1024) with both collectives as peer kernels over an emulated
    group: stats all-gather == torch.stack of the ranks' stats (bytes), summed partials identical on
    every rank and == the rank-order sum, merged indices == the unsharded run, oracle parity on a unit."""
    n, S, B, H, Hkv, d = 524288, 1024, 1, 32, 8, 128
    inp = si.make_decode_inputs(B, H, Hkv, d, n, dtype="bf16", seed=45, device="cuda")
    full_idx = santa.decode(inp.q, inp.K, inp.V, inp.seqlens, S, "stratified", 7, 3, return_idx=True)[1]
    bounds = sharding.shard_bounds(n, R)
    grp = sharding.EmulatedPeerGroup(R, B * H * d * 4)
    stats, shards = [], []
    for r in range(R):
        a, e = bounds[r]
        sl = torch.tensor([e - a], dtype=torch.int32, device="cuda")
        be = sharding.CudaBackend()
        stats.append(be.stats(inp.q, inp.K[:, :, a:e].contiguous(), sl, Hkv, S))
        shards.append((be, inp.V[:, :, a:e].contiguous(), sl, torch.tensor([a], dtype=torch.int32, device="cuda")))
    gathered = grp.all_gather(stats)
    torch.cuda.synchronize()
    ref_all = torch.stack(stats, 0)
    assert all(torch.equal(g, ref_all) for g in gathered)
    parts, merged = [], torch.full((B, H, S), -1, dtype=torch.int32, device="cuda")
    for r, (be, Vs, sl, off) in enumerate(shards):
        part, idx = be.sample_gather(gathered[r], r, R, off, Vs, sl, S, "stratified", 7, 3, return_idx=True)
        parts.append(part)
        merged = torch.where(idx >= 0, idx, merged)
    ref_sum = parts[0].clone()
    for p in parts[1:]:
        ref_sum = ref_sum + p
    grp.all_reduce_(parts)
    torch.cuda.synchronize()
    assert all(torch.equal(p, ref_sum) for p in parts)
    assert (merged != full_idx).float().mean().item() < 1e-3
    tot, mis = unit_parity(inp, parts[0].to(torch.bfloat16), merged, [(0, 5)], S, "stratified", 7, 3)
    print(f"config 4 R={R} over the peer exchange: {mis}/{tot} index mismatches vs the oracle")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _ipc_worker(rank, world, port, q):
    """Rank 1 exports its exchange buffer; rank 0 maps it (CUDA IPC) and serves BOTH ranks in one
    emulated launch: its writes land in rank 1's allocation and its reads of rank 1's slots come back
    through the mapping.  Rank 1 then finds the pushed slots and flags in its own memory."""
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2605_01910_b200 as sa
        nbytes = sa.santa_peer_buffer_bytes(2, 4096)
        own = torch.zeros(nbytes + 512, dtype=torch.uint8, device="cuda")[512:]   # non-zero offset in its allocation
        torch.cuda.synchronize()
        handles = [None, None]
        dist.all_gather_object(handles, sa.santa_ipc_export(own))
        if rank == 0:
            p1, base = sa.santa_ipc_import(*handles[1])
            grp = sa.make_peer_group([own.data_ptr(), p1], nbytes)
            src = [torch.arange(1024, dtype=torch.float32, device="cuda") * (r + 1) for r in range(2)]
            dst = [torch.empty(1024, device="cuda") for _ in range(2)]
            sa.santa_peer_allreduce_f32(grp, [0, 1], src, dst, 1)
            torch.cuda.synchronize()
            want = torch.arange(1024, dtype=torch.float32, device="cuda") * 3
            assert torch.equal(dst[0], want) and torch.equal(dst[1], want)
        dist.barrier()
        if rank == 1:
            # epoch 1 -> parity 1; slot of source 0 holds rank 0's payload; flag[1][src][0] == 1
            flags = own[256:256 + 4096].view(torch.int32).view(2, 8, 64)
            assert int(flags[1, 0, 0]) == 1 and int(flags[1, 1, 0]) == 1 and int(flags[0].abs().sum()) == 0
            slot = (nbytes - 8192) // 4
            data = own[8192:].view(torch.float32)
            s0 = data[(2 + 0) * slot // 4:(2 + 0) * slot // 4 + 1024]
            assert torch.equal(s0, torch.arange(1024, dtype=torch.float32, device="cuda"))
        dist.barrier()
        if rank == 0:
            sa.santa_ipc_close(base)
        q.put("ok")
    except Exception as e:
        q.put(repr(e))
        raise
    finally:
        dist.destroy_process_group()


def test_ipc_mapping_two_processes():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    mp.start_processes(_ipc_worker, args=(2, _free_port(), q), nprocs=2, join=True, start_method="spawn")
    for _ in range(2):
        r = q.get(timeout=5)
        assert r == "ok", r


def _peer_exchange_worker(rank, world, port, q):
    """sharding.PeerExchange built by two processes on one GPU (export, all_gather_object of the
    handles, import, the all-ranks success vote): every rank sees both buffers; rank 0 then pushes one
    emulated all-gather through rank 1's mapping (no kernel waits on another process) and rank 1 finds
    the flags in its own buffer; close() unmaps."""
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2605_01910_b200 as sa
        from paper_2605_01910_b200 import sharding as sh
        ex = sh.PeerExchange(1024, device="cuda")
        assert ex.world == 2 and ex.peer_group.world == 2
        assert ex.peer_group.bufs[rank] == ex.buf.data_ptr()
        if rank == 0:
            src = [torch.full((256,), float(r + 1), device="cuda") for r in range(2)]
            dst = [torch.empty(2 * 256, device="cuda") for _ in range(2)]
            sa.santa_peer_allgather(ex.peer_group, [0, 1], src, dst, 1)
            torch.cuda.synchronize()
            assert torch.equal(dst[1][:256], src[0]) and torch.equal(dst[1][256:], src[1])
        dist.barrier()
        if rank == 1:
            flags = ex.buf[256:256 + 4096].view(torch.int32).view(2, 8, 64)
            assert int(flags[1, 0, 0]) == 1 and int(flags[1, 1, 0]) == 1
        ex.close()
        q.put("ok")
    except Exception as e:
        q.put(repr(e))
        raise
    finally:
        dist.destroy_process_group()


def test_peer_exchange_class_two_processes():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    mp.start_processes(_peer_exchange_worker, args=(2, _free_port(), q), nprocs=2, join=True, start_method="spawn")
    for _ in range(2):
        r = q.get(timeout=5)
        assert r == "ok", r
