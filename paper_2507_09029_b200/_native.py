"""ctypes binding of libsdp.so (include/sdp.h).

The product path has no CPU fallback: if the library is missing or the CUDA
device is unavailable, every entry point raises.  `lib()` loads the in-tree
build (paper_2507_09029_b200/_lib/libsdp.so); run
`python -m paper_2507_09029_b200.build` (or __graft_entry__.build()) first.
"""

from __future__ import annotations

import ctypes as C
import threading
from pathlib import Path

from .errors import STATUS_CLASSES, NativeLibraryMissing, SubnetError

LIB_PATH = Path(__file__).resolve().parent / "_lib" / "libsdp.so"
ABI_VERSION = 2
MAX_WORKERS = 64

# status words (SDP_STATUS_*)
STATUS_UNCOVERED_LEAK = 0x1
STATUS_NONFINITE = 0x2
STATUS_BARRIER_TIMEOUT = 0x4

# sync flags (SDP_SYNC_*)
SYNC_WRITEBACK = 0x1
SYNC_CHECK_UNCOVERED = 0x2
SYNC_CHECK_FINITE = 0x4
SYNC_NESTEROV = 0x8
SYNC_ADAM = 0x10
SYNC_LOCAL_UPDATE = 0x20
SYNC_DIRECT = 0x40
SYNC_STREAM = 0x80

SCATTER_ZERO_FILL = 0x1
SCATTER_ACCUMULATE = 0x2

DTYPE_F32 = 0
DTYPE_F64 = 1
DTYPE_U8 = 2
DTYPE_U16 = 3
GATHER_REVERSE = 0x1

TILE_UNIFORM = 0x80000000
TILE_LEN_MASK = 0x00FFFFFF


class GroupDesc(C.Structure):
    _fields_ = [("first_unit", C.c_int32), ("size", C.c_int32)]


class ParamDesc(C.Structure):
    _fields_ = [("offset", C.c_int64), ("size", C.c_int64),
                ("rule_begin", C.c_int32), ("rule_count", C.c_int32)]


class RuleDesc(C.Structure):
    _fields_ = [("inner", C.c_int32), ("dim", C.c_int32), ("unit_base", C.c_int32),
                ("inner_mul", C.c_uint32), ("inner_shr", C.c_uint32),
                ("dim_mul", C.c_uint32), ("dim_shr", C.c_uint32), ("pad_", C.c_int32)]


class TileDesc(C.Structure):
    _fields_ = [("owner_bits", C.c_uint64), ("tile_index", C.c_uint32),
                ("len_flags", C.c_uint32)]


class SliceDesc(C.Structure):
    _fields_ = [("full_offset", C.c_int64), ("compact_offset", C.c_int64),
                ("rows", C.c_int32), ("cols", C.c_int32), ("inner", C.c_int32),
                ("crows", C.c_int32), ("ccols", C.c_int32),
                ("row_map", C.c_int32), ("col_map", C.c_int32),
                ("inner_mul", C.c_uint32), ("inner_shr", C.c_uint32),
                ("rowlen_mul", C.c_uint32), ("rowlen_shr", C.c_uint32), ("col_tab", C.c_int32)]


class SliceTask(C.Structure):
    _fields_ = [("desc", C.c_int32), ("row_begin", C.c_int32), ("row_end", C.c_int32),
                ("elem_begin", C.c_int32), ("elem_end", C.c_int32), ("seg", C.c_int32),
                ("pad_", C.c_int32 * 2)]


class SliceSegs(C.Structure):
    _fields_ = [("full", C.c_void_p * MAX_WORKERS), ("compact", C.c_void_p * MAX_WORKERS), ("n", C.c_int32)]



class SyncArgs(C.Structure):
    _fields_ = [
        ("dtype", C.c_int32), ("n_workers", C.c_int32), ("mask_bytes", C.c_int32),
        ("tile", C.c_int32), ("total", C.c_int64),
        ("owner_mask", C.c_void_p), ("tiles", C.c_void_p),
        ("n_tiles", C.c_int32), ("tiles_per_cta", C.c_int32), ("grid", C.c_int32),
        ("flags", C.c_int32),
        ("replicas", C.c_void_p * MAX_WORKERS), ("shadow_bf16", C.c_void_p * MAX_WORKERS),
        ("out", C.c_void_p), ("out_bf16", C.c_void_p),
        ("theta", C.c_void_p), ("velocity", C.c_void_p), ("theta_bf16", C.c_void_p),
        ("lr", C.c_double), ("momentum", C.c_double),
        ("status", C.c_void_p),
        ("rank", C.c_int32), ("world", C.c_int32),
        ("signal_pads", C.c_void_p * 8),
        ("epoch", C.c_uint32), ("pad_", C.c_uint32),
        ("timeout_cycles", C.c_int64),
        ("second_moment", C.c_void_p),
        ("beta1", C.c_double), ("beta2", C.c_double), ("one_minus_beta1", C.c_double),
        ("one_minus_beta2", C.c_double), ("bias1", C.c_double), ("bias2", C.c_double),
        ("eps", C.c_double),
        ("epoch_counters", C.c_void_p),
        ("slots", C.c_void_p), ("slot_stride", C.c_int64),
        ("updates", C.c_void_p), ("updates_per_cta", C.c_int32), ("pad2_", C.c_int32),
        ("states", C.c_void_p),
        ("adam_step", C.c_void_p), ("adam_bias_table", C.c_void_p), ("adam_table_len", C.c_int32),
        ("pad3_", C.c_int32),
    ]


class WorkerState(C.Structure):
    _fields_ = [("theta", C.c_void_p), ("velocity", C.c_void_p), ("second_moment", C.c_void_p),
                ("theta_bf16", C.c_void_p), ("grad", C.c_void_p)]


class UpdateDesc(C.Structure):
    _fields_ = [("state", C.c_uint32), ("slot", C.c_uint32), ("len", C.c_uint32), ("pad_", C.c_uint32)]


VP, I32, I64, U64, DBL = C.c_void_p, C.c_int, C.c_int64, C.c_uint64, C.c_double

# name -> (restype, argtypes); every exported symbol of include/sdp.h
SIGNATURES = {
    "sdp_abi_version": (C.c_int, []),
    "sdp_last_error": (C.c_char_p, []),
    "sdp_device_sm_count": (C.c_int, [C.POINTER(C.c_int)]),
    "sdp_host_ptr_on_device": (C.c_int, [VP, C.POINTER(C.c_int)]),
    "sdp_ce_rows_fwd": (C.c_int, [VP, I64, I32, I64, VP, VP, VP, VP]),
    "sdp_group_norm_fwd": (C.c_int, [VP, I32, I32, I32, VP, I32, I32, VP, VP, C.c_float, I32, VP, VP, VP, VP]),
    "sdp_group_norm_bwd_scratch": (C.c_int, [I32, I32, I32, I32, C.POINTER(C.c_longlong)]),
    "sdp_group_norm_bwd": (C.c_int, [VP, VP, VP, I32, I32, I32, VP, I32, I32, VP, VP, VP, I32, VP, VP, VP, VP,
                                     C.c_longlong, VP]),
    "sdp_layer_norm_fwd": (C.c_int, [VP, I64, I32, VP, VP, C.c_float, VP, VP, VP, VP]),
    "sdp_layer_norm_bwd_parts": (C.c_int, [I64, I32]),
    "sdp_layer_norm_bwd": (C.c_int, [VP, VP, I64, I32, VP, VP, VP, VP, VP, VP, VP, I32, VP]),
    "sdp_add_layer_norm_fwd": (C.c_int, [VP, VP, I64, I32, VP, VP, C.c_float, VP, VP, VP, VP, VP]),
    "sdp_layer_norm_bwd_res": (C.c_int, [VP, VP, VP, I64, I32, VP, VP, VP, VP, VP, VP, VP, I32, VP]),
    "sdp_merge_heads": (C.c_int, [VP, VP, VP, I64, I64, I32, I32, I32, I64, I64, I64, VP, VP]),
    "sdp_conv_grads_to_oihw": (C.c_int, [VP, I32, I32, VP, VP, VP]),
    "sdp_conv_grad_max_block": (C.c_int, []),
    "sdp_conv_weights_to_ohwi": (C.c_int, [VP, I32, I32, VP, VP, VP]),
    "sdp_col_sum_parts": (C.c_int, []),
    "sdp_col_sum_bf16": (C.c_int, [VP, I64, I32, VP, VP, VP]),
    "sdp_ce_rows_bwd": (C.c_int, [VP, I64, I32, I64, VP, VP, VP, C.c_float, VP, VP]),
    "sdp_assign_units": (C.c_int, [C.POINTER(C.c_uint32), I32, VP, I32, I32, I32, I32, I32, VP, VP, VP]),
    "sdp_permutation": (C.c_int, [C.POINTER(C.c_uint32), I32, VP, I32, I32, VP, VP]),
    "sdp_build_masks": (C.c_int, [VP, I32, VP, I32, VP, I32, I64, VP, I32, VP, VP, VP, VP, VP, VP]),
    "sdp_worker_mask": (C.c_int, [VP, I32, I64, I32, VP, VP, VP]),
    "sdp_plan_tiles": (C.c_int, [VP, I32, I64, I32, VP, VP, VP]),
    "sdp_owner_sync": (C.c_int, [C.POINTER(SyncArgs), VP]),
    "sdp_nesterov_update": (C.c_int, [I32, I64, VP, VP, VP, DBL, DBL, VP, VP, VP]),
    "sdp_adam_update": (C.c_int, [I32, I64, VP, VP, VP, VP, DBL, DBL, DBL, DBL, I32, VP, VP]),
    "sdp_check_finite": (C.c_int, [I32, I64, VP, VP, VP]),
    "sdp_masked_extract": (C.c_int, [I32, VP, VP, I32, I64, I32, VP, VP]),
    "sdp_gather_slices": (C.c_int, [I32, VP, VP, I32, VP, VP, VP, I32, VP]),
    "sdp_scatter_slices": (C.c_int, [I32, VP, VP, I32, VP, VP, VP, I32, VP]),
    "sdp_gather_slices_multi": (C.c_int, [I32, VP, VP, I32, VP, C.POINTER(SliceSegs), I32, VP]),
    "sdp_scatter_slices_multi": (C.c_int, [I32, VP, VP, I32, VP, C.POINTER(SliceSegs), I32, VP]),
    "sdp_divide": (C.c_int, [I32, VP, VP, I64, VP, VP]),
    "sdp_restricted_dots": (C.c_int, [I32, VP, VP, VP, VP, I32, I32, VP, VP, VP]),
    "sdp_ipc_export": (C.c_int, [VP, C.POINTER(C.c_uint8), C.POINTER(C.c_uint64)]),
    "sdp_ipc_import": (C.c_int, [C.POINTER(C.c_uint8), C.c_uint64, C.POINTER(C.c_void_p)]),
    "sdp_ipc_close": (C.c_int, [VP]),
    "sdp_enable_peer": (C.c_int, [I32]),
    "sdp_copy_async": (C.c_int, [VP, VP, C.c_size_t, VP]),
}

_lock = threading.Lock()
_lib: C.CDLL | None = None


def load(path: Path | str = LIB_PATH) -> C.CDLL:
    """Load libsdp.so and bind every symbol (no device work happens here)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        p = Path(path)
        if not p.exists():
            raise NativeLibraryMissing(
                f"{p} is missing: build it with `python -m paper_2507_09029_b200.build`; "
                "there is no CPU fallback for the subnetwork-DP hot path")
        try:
            lib = C.CDLL(str(p), mode=C.RTLD_GLOBAL)
        except OSError as exc:
            raise NativeLibraryMissing(f"cannot load {p}: {exc}") from exc
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.sdp_abi_version() != ABI_VERSION:
            raise NativeLibraryMissing(
                f"{p} has ABI {lib.sdp_abi_version()}, expected {ABI_VERSION}; rebuild it")
        _lib = lib
        return lib


def lib() -> C.CDLL:
    return _lib if _lib is not None else load()


def check(rc: int, what: str = "") -> None:
    """Raise the reference exception class that status `rc` maps to."""
    if rc == 0:
        return
    msg = lib().sdp_last_error().decode(errors="replace")
    cls = STATUS_CLASSES.get(rc, SubnetError)
    raise cls(f"{what}: {msg}" if what else msg)


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args), name)


def seed_words(seed: int) -> tuple[C.Array, int]:
    """Non-negative seed -> little-endian uint32 words (SeedSequence entropy)."""
    seed = int(seed)
    if seed < 0:
        raise ValueError("seed must be non-negative")
    words = []
    while True:
        words.append(seed & 0xFFFFFFFF)
        seed >>= 32
        if not seed:
            break
    if len(words) > 8:
        raise ValueError("seeds above 2**256 are not supported")
    arr = (C.c_uint32 * len(words))(*words)
    return arr, len(words)
