"""ctypes binding of libsanta.so (include/santa.h).  Argument marshalling only: every step
of the decode path runs in the CUDA kernels behind these calls.  PyTorch is used for
device memory, streams and nothing else.  If the library is missing, importing this
module raises -- there is no fallback."""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SANTA_LIB_PATH") or os.path.join(_HERE, "_lib", "libsanta.so")  # override: A/B builds (tools/)

SANTA_OK = 0
STATUS = {0: "SANTA_OK", 1: "SANTA_ERR_INVALID_ARG", 2: "SANTA_ERR_SHAPE", 3: "SANTA_ERR_EMPTY_BUDGET",
          4: "SANTA_ERR_EMPTY_DISTRIBUTION", 5: "SANTA_ERR_UNSUPPORTED", 6: "SANTA_ERR_WORKSPACE",
          7: "SANTA_ERR_ALIGNMENT", 8: "SANTA_ERR_CUDA"}
MODES = {"iid": 0, "stratified": 1, "systematic": 2}
DTYPES = {"bf16": 0, "f32": 1, "f16": 2}
FLAG_EMPTY_SEQ = 0x1
FLAG_SYNC_TIMEOUT = 0x100
FLAG_PEER_TIMEOUT = 0x200
IPC_HANDLE_BYTES = 64
PATHS = {"auto": 0, "step": 1, "two_kernel": 2, "step_tc": 3}


class SantaError(RuntimeError):
    def __init__(self, fn: str, status: int):
        super().__init__(f"{fn} failed: {STATUS.get(status, status)}")
        self.status = status


class LayerSchedule(ctypes.Structure):
    _fields_ = [("n_layers", ctypes.c_int32), ("S", ctypes.POINTER(ctypes.c_int32))]


class Geometry(ctypes.Structure):
    _fields_ = [
        ("batch", ctypes.c_int32),
        ("n_heads", ctypes.c_int32),
        ("n_kv_heads", ctypes.c_int32),
        ("head_dim", ctypes.c_int32),
        ("dtype", ctypes.c_int32),
        ("page_size", ctypes.c_int32),
        ("max_pages_per_seq", ctypes.c_int32),
        ("page_table", ctypes.c_void_p),
        ("max_seqlen", ctypes.c_int32),
        ("scale", ctypes.c_float),
        ("batch_offset", ctypes.c_int32),
        ("head_offset", ctypes.c_int32),
    ]


class PeerGroup(ctypes.Structure):
    _fields_ = [("world", ctypes.c_int32), ("bufs", ctypes.c_void_p * 8), ("buf_bytes", ctypes.c_size_t)]


def _load() -> ctypes.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libsanta.so not built ({LIB_PATH}); run `make` or __graft_entry__.build()")
    lib = ctypes.CDLL(LIB_PATH)
    vp, i32, u64, sz = ctypes.c_void_p, ctypes.c_int32, ctypes.c_uint64, ctypes.c_size_t
    G = ctypes.POINTER(Geometry)
    sigs = {
        "santa_status_string": ([i32], ctypes.c_char_p),
        "santa_version": ([], ctypes.c_char_p),
        "santa_workspace_bytes": ([G, i32], sz),
        "santa_auto_path": ([G, i32], i32),
        "santa_decode_attention": ([G, vp, vp, vp, vp, i32, i32, u64, u64, vp, vp, vp, sz, vp], i32),
        "santa_decode_attention_path": ([G, vp, vp, vp, vp, i32, i32, u64, u64, vp, vp, vp, sz, i32, vp], i32),
        "santa_decode_attention_profiled": ([G, vp, vp, vp, vp, i32, i32, u64, u64, vp, vp, vp, sz, vp, vp], i32),
        "santa_dense_reference": ([G, vp, vp, vp, vp, vp, vp, sz, vp], i32),
        "santa_decode_attention_prop": ([G, vp, vp, vp, vp, i32, u64, u64, vp, vp, vp, sz, vp], i32),
        "santa_prop_tile_len": ([G], i32),
        "santa_decode_attention_flash": ([G, vp, vp, vp, vp, i32, i32, u64, u64, vp, vp, vp, sz, vp], i32),
        "santa_flash_max_samples": ([G, i32, i32], i32),
        "santa_score_phase": ([G, vp, vp, vp, vp, sz, vp], i32),
        "santa_sample_phase": ([G, vp, vp, i32, i32, u64, u64, vp, vp, vp, sz, vp], i32),
        "santa_bernoulli_scores": ([G, vp, vp, vp, i32, i32, i32, u64, u64, vp, vp, vp, sz, vp], i32),
        "santa_decode_attention_bernoulli": ([G, vp, vp, vp, vp, i32, i32, i32, i32, i32, u64, u64, vp, vp, vp,
                                              sz, vp], i32),
        "santa_seqshard_stats": ([G, vp, vp, vp, vp, vp, sz, vp], i32),
        "santa_seqshard_sample_gather": ([G, vp, i32, i32, vp, vp, vp, i32, i32, u64, u64, vp, vp, vp, sz, vp],
                                         i32),
        "santa_decode_step_host": ([G, vp, vp, vp, vp, vp, vp, vp, vp, vp, i32, i32, u64, u64, vp, vp, vp, sz,
                                    vp], i32),
        "santa_decode_step_host_packed": ([G, vp, vp, vp, vp, vp, i32, i32, u64, u64, vp, vp, vp, sz, i32, vp], i32),
        "santa_philox_uniforms": ([u64, u64, i32, i32, i32, i32, vp, vp, vp, vp], i32),
        "santa_read_error_flags": ([vp, ctypes.POINTER(ctypes.c_uint32), vp], i32),
        "santa_decode_attention_append": ([G, vp, vp, vp, vp, vp, vp, i32, i32, u64, u64, vp, vp, vp, sz, vp], i32),
        "santa_schedule_workspace_bytes": ([G, ctypes.POINTER(LayerSchedule)], sz),
        "santa_decode_attention_layer": ([G, ctypes.POINTER(LayerSchedule), i32, vp, vp, vp, vp, vp, vp, i32, u64,
                                          u64, vp, vp, vp, sz, vp], i32),
        "santa_peer_buffer_bytes": ([i32, sz], sz),
        "santa_peer_allgather": ([ctypes.POINTER(PeerGroup), i32, vp, vp, vp, sz, ctypes.c_uint32, vp], i32),
        "santa_peer_allreduce_f32": ([ctypes.POINTER(PeerGroup), i32, vp, vp, vp, sz, ctypes.c_uint32, vp], i32),
        "santa_ipc_export": ([vp, vp, ctypes.POINTER(sz)], i32),
        "santa_ipc_import": ([vp, sz, ctypes.POINTER(vp), ctypes.POINTER(vp)], i32),
        "santa_ipc_close": ([vp], i32),
    }
    for name, (args, res) in sigs.items():
        if os.environ.get("SANTA_LIB_PATH") and not hasattr(lib, name):
            continue  # A/B timing against an older build (tools only)
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = res
    return lib


LIB = _load()


def check(fn: str, status: int) -> None:
    if status != SANTA_OK:
        raise SantaError(fn, status)
