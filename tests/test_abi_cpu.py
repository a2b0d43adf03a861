"""C-ABI checks that need no GPU (-m "not gpu"): the library loads, exports every symbol
include/santa.h declares, sizes its workspace by pure host arithmetic, and rejects invalid
arguments before touching CUDA."""
import ctypes
import os
import re

import pytest
import torch

from conftest import ROOT

import paper_2605_01910_b200 as santa
from paper_2605_01910_b200 import _abi


def _declared():
    src = open(os.path.join(ROOT, "include", "santa.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(santa_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    names = _declared()
    assert len(names) >= 13
    for n in names:
        assert hasattr(_abi.LIB, n), n


def test_library_is_sm100a_only():
    out = os.popen(f"cuobjdump -lelf {santa.LIB_PATH} 2>&1").read()
    assert "sm_100a" in out and "sm_90" not in out.replace("sm_100a", "")
    assert "sm_100a" in santa.santa_version()


def test_status_strings():
    for code, name in _abi.STATUS.items():
        assert _abi.LIB.santa_status_string(code).decode() == name


def _geo(**kw):
    g = _abi.Geometry()
    g.batch, g.n_heads, g.n_kv_heads, g.head_dim, g.dtype = 1, 32, 8, 128, 0
    g.max_seqlen, g.scale = 32768, 0.0
    for k, v in kw.items():
        setattr(g, k, v)
    return g


def test_workspace_bytes_host_arithmetic():
    g = _geo()
    n = santa.santa_workspace_bytes(g, 256)
    C = 32768 // 256
    stash = 32 * C * 256 * 4
    assert stash < n < 3 * stash            # stash + Bernoulli score scratch + small tables
    assert santa.santa_workspace_bytes(_geo(n_heads=30), 256) == 0     # H % H_kv
    assert santa.santa_workspace_bytes(_geo(head_dim=96), 256) == 0    # unsupported d
    assert santa.santa_workspace_bytes(_geo(max_seqlen=0), 256) == 0
    assert santa.santa_workspace_bytes(g, 0) == 0
    assert santa.santa_workspace_bytes(_geo(n_heads=128, n_kv_heads=8), 1) == 0   # G = 16


@pytest.mark.parametrize("kw,status", [
    (dict(n_heads=30), 2), (dict(head_dim=80), 5), (dict(max_seqlen=0), 4), (dict(dtype=9), 1),
    (dict(batch=0), 2), (dict(n_heads=64, n_kv_heads=4), 5), (dict(scale=float("nan")), 1),
    (dict(page_table=16, page_size=24, max_pages_per_seq=4096), 2),
])
def test_invalid_geometry_rejected_without_gpu(kw, status):
    g = _geo(**kw)
    st = _abi.LIB.santa_decode_attention(ctypes.byref(g), 16, 16, 16, 16, 256, 1, 0, 0, 16, None, 256, 1 << 30, None)
    assert st == status


def test_invalid_call_arguments_rejected_without_gpu():
    g = _geo()
    L = _abi.LIB
    assert L.santa_decode_attention(ctypes.byref(g), 16, 16, 16, 16, 0, 1, 0, 0, 16, None, 256, 1 << 30, None) == 3
    assert L.santa_decode_attention(ctypes.byref(g), 16, 16, 16, 16, 8, 5, 0, 0, 16, None, 256, 1 << 30, None) == 1
    assert L.santa_decode_attention(ctypes.byref(g), None, 16, 16, 16, 8, 1, 0, 0, 16, None, 256, 1 << 30, None) == 1
    assert L.santa_decode_attention(ctypes.byref(g), 8, 16, 16, 16, 8, 1, 0, 0, 16, None, 256, 1 << 30, None) == 7
    assert L.santa_decode_attention(ctypes.byref(g), 16, 16, 16, 16, 8, 1, 0, 0, 16, None, 128, 1 << 30, None) == 6
    assert L.santa_decode_attention(ctypes.byref(g), 16, 16, 16, 16, 8, 1, 0, 0, 16, None, 256, 1000, None) == 6
    assert L.santa_bernoulli_scores(ctypes.byref(g), 16, 16, 16, 0, 1, 1, 0, 0, 16, None, 256, 1 << 30, None) == 3
    assert L.santa_seqshard_sample_gather(ctypes.byref(g), 16, 2, 2, 16, 16, 16, 8, 1, 0, 0, 16, None, 256,
                                          1 << 30, None) == 1
    assert L.santa_philox_uniforms(0, 0, 1, 0, 0, 0, 16, None, None, None) == 1


def test_binding_refuses_cpu_tensors():
    q = torch.zeros(1, 4, 128, dtype=torch.bfloat16)
    K = torch.zeros(1, 1, 16, 128, dtype=torch.bfloat16)
    with pytest.raises(ValueError):
        santa.decode(q, K, K, torch.tensor([16], dtype=torch.int32), 4, ws=torch.zeros(1 << 20, dtype=torch.uint8))


def test_product_package_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_2605_01910_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(from|import)\s+oracle|santa_oracle|oracle\.", txt, re.M), f


def test_auto_path_policy_is_host_logic():
    """santa_auto_path (pure host arithmetic): the two-kernel path for every geometry since round 2
    (profiles/r02/v95_path_sweep_step_pdl.txt)."""
    assert santa.santa_auto_path(_geo(), 256) == "two_kernel"             # config 2
    assert santa.santa_auto_path(_geo(batch=32), 64) == "two_kernel"      # config 3, S = 64
    assert santa.santa_auto_path(_geo(batch=32), 256) == "two_kernel"     # config 3, S = 256
    assert santa.santa_auto_path(_geo(batch=32), 512) == "two_kernel"
    assert santa.santa_auto_path(_geo(batch=32), 1024) == "two_kernel"
    assert santa.santa_auto_path(_geo(batch=32, dtype=1), 256) == "two_kernel"   # fp32 cache
    assert santa.santa_auto_path(_geo(batch=32, max_seqlen=131072), 256) == "two_kernel"
    with pytest.raises(santa.SantaError):
        santa.santa_auto_path(_geo(max_seqlen=0), 256)


def test_prop_and_flash_host_logic():
    """S^2ANTA-prop / -flash entry points: tile length, flash idx row length (max over sequence lengths
    of S_tile * T, against the oracle's S_tile rule) and argument rejection -- all before any launch."""
    from oracle import santa_oracle as o
    L = _abi.LIB
    for n, tile in ((32768, 64), (524288, 64), (524289, 128), (1 << 20, 128)):
        g = _geo(max_seqlen=n)
        assert L.santa_prop_tile_len(ctypes.byref(g)) == tile
    g = _geo(max_seqlen=32768)
    for S, tile in ((2048, 256), (256, 64), (1, 1024), (7, 128)):
        want = max(o.flash_tile_budget(T * tile, tile, S) * T for T in range(1, 32768 // tile + 1))
        assert L.santa_flash_max_samples(ctypes.byref(g), S, tile) == want
    for bad in (0, 32, 96, 64 * 65):
        assert L.santa_flash_max_samples(ctypes.byref(g), 64, bad) == -1
    a = (16, 16, 16, 16)
    assert L.santa_decode_attention_prop(ctypes.byref(g), *a, 0, 0, 0, 16, None, 256, 1 << 30, None) == 3
    assert L.santa_decode_attention_prop(ctypes.byref(g), None, 16, 16, 16, 8, 0, 0, 16, None, 256, 1 << 30,
                                         None) == 1
    assert L.santa_decode_attention_flash(ctypes.byref(g), *a, 8, 100, 0, 0, 16, None, 256, 1 << 30, None) == 1
    assert L.santa_decode_attention_flash(ctypes.byref(g), *a, 0, 256, 0, 0, 16, None, 256, 1 << 30, None) == 3


def test_wrappers_refuse_mismatched_cache_shapes():
    """for a contiguous cache the row stride of K/V IS max_seqlen; the convenience
    wrappers refuse a max_seqlen different from K.shape[2], K/V shape or dtype mismatches and a
    malformed paged pool -- before any CUDA call (these are CPU tensors)."""
    B, H, Hkv, n, d = 2, 8, 2, 256, 64
    q = torch.zeros(B, H, d, dtype=torch.bfloat16)
    K = torch.zeros(B, Hkv, n, d, dtype=torch.bfloat16)
    V = torch.zeros_like(K)
    sl = torch.full((B,), n, dtype=torch.int32)
    for fn in (lambda **kw: santa.decode(q, K, V, sl, 16, **kw),
               lambda **kw: santa.decode_prop(q, K, V, sl, 16, **kw),
               lambda **kw: santa.decode_flash(q, K, V, sl, 16, 64, **kw),
               lambda **kw: santa.dense(q, K, V, sl, **kw)):
        with pytest.raises(ValueError, match="max_seqlen"):
            fn(max_seqlen=128)                       # smaller than the row stride
    with pytest.raises(ValueError, match="dtype"):
        santa.decode(q, K, V.float(), sl, 16)
    with pytest.raises(ValueError, match="shapes differ"):
        santa.decode(q, K, V[:, :, :128], sl, 16)
    with pytest.raises(ValueError, match="H_kv"):
        santa.decode(q, K[:, :1], V[:, :1], sl, 16, n_kv_heads=2)
    pool = torch.zeros(8, Hkv, 64, d, dtype=torch.bfloat16)
    pt = torch.zeros(B, 4, dtype=torch.int64)
    with pytest.raises(ValueError, match="page_table"):
        santa.decode(q, pool, pool, sl, 16, page_table=pt, page_size=64)
    with pytest.raises(ValueError, match="paged pool"):
        santa.decode(q, pool, pool, sl, 16, page_table=pt.int(), page_size=32)


def test_layer_schedule_host_logic():
    """Per-layer budgets (App. K): the schedule's workspace is the max over its layers' workspaces;
    malformed schedules are refused (0 bytes) without a GPU."""
    g = _geo()
    sched = santa.make_schedule([8, 256, 64, 1024])
    want = max(santa.santa_workspace_bytes(g, S) for S in (8, 256, 64, 1024))
    assert santa.santa_schedule_workspace_bytes(g, sched) == want
    assert santa.santa_schedule_workspace_bytes(g, santa.make_schedule([8, 0])) == 0       # S < 1
    assert santa.santa_schedule_workspace_bytes(g, santa.make_schedule([8, 5000])) == 0    # S > 4096
    assert santa.santa_schedule_workspace_bytes(_geo(head_dim=96), sched) == 0


def test_peer_exchange_host_checks():
    """santa_peer_* (config 4's one-shot exchange): buffer arithmetic and argument checks need no GPU."""
    assert santa.santa_peer_buffer_bytes(2, 512) == 8192 + 2 * 2 * 512
    assert santa.santa_peer_buffer_bytes(8, 100) == 8192 + 2 * 8 * 256     # slots rounded to 256 B
    assert santa.santa_peer_buffer_bytes(0, 512) == 0
    assert santa.santa_peer_buffer_bytes(9, 512) == 0
    g = santa.make_peer_group([0x10000, 0x20000], santa.santa_peer_buffer_bytes(2, 4096))
    ranks = (ctypes.c_int32 * 2)(0, 1)
    ptrs = (ctypes.c_void_p * 2)(0x30000, 0x40000)
    call = lambda **kw: _abi.LIB.santa_peer_allgather(  # noqa: E731
        ctypes.byref(kw.get("g", g)), kw.get("n", 2), kw.get("ranks", ranks), ptrs, ptrs, kw.get("nb", 4096),
        kw.get("epoch", 1), None)
    assert call(epoch=0) == 1                       # INVALID_ARG
    assert call(n=3) == 1                           # more local ranks than the group
    assert call(ranks=(ctypes.c_int32 * 2)(1, 1)) == 1
    assert call(nb=4100) == 7                       # ALIGNMENT: payload not a multiple of 16
    assert call(nb=8192) == 6                       # WORKSPACE: payload larger than a slot
    g2 = santa.make_peer_group([0x10000, 0x20010], g.buf_bytes)
    assert call(g=g2) == 7                          # buffer not 256-B aligned
    g9 = santa.make_peer_group([0x10000] * 8, g.buf_bytes)
    g9.world = 9
    assert call(g=g9) == 1
