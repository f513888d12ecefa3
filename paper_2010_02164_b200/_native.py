"""ctypes binding of the C-ABI in include/varstream.h (libvarstream.so, sm_100a).

The library is built in-tree by ``__graft_entry__.build()`` (nvcc, no torch
types in any signature).  There is no CPU fallback: importing the engine on a
machine without the library or without a CUDA device raises immediately.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

from .errors import ConfigError, InvariantViolation

LIB_PATH = Path(__file__).resolve().parent / "_lib" / "libvarstream.so"

VS_OK, VS_ERR_CONFIG, VS_ERR_INVARIANT, VS_ERR_CUDA = 0, -1, -3, -4
VS_DTYPE_F32, VS_DTYPE_BF16, VS_DTYPE_F64, VS_ROWS_NORMALIZED = 0, 1, 2, 0x100
VS_K1_SPLIT, VS_K1_WARP = 0x200, 0x400  # pin the K1 kernel (vs_row_lse_topm_ws)
# BatchedScorer.logits may return this code: the scorer already produced K1's
# outputs (top_tok / top_logp / row_lse) for the step, e.g. with the fused K5 head
VS_K1_DONE = -1
VS_POLICY_DEFERRED, VS_POLICY_IMMEDIATE = 0, 1
VS_ADMIT_NONE, VS_ADMIT_VARSTREAM, VS_ADMIT_VARBEAM, VS_ADMIT_VARFIFO = -1, 0, 1, 2
VS_SELECT_MIN_LT, VS_SELECT_FIFO, VS_SELECT_ALL = 0, 1, 2
VS_MAX_K, VS_MAX_M, VS_MAX_SLOTS = 128, 128, 1024

ST_R, ST_NSEL, ST_NLIVE, ST_L, ST_NADMIT, ST_ADMIT0, ST_CURSOR, ST_DONE = range(8)
ST_ERROR, ST_NFIN, ST_NLIVE_AFTER, ST_TOKFILL, ST_MINLIVE = 8, 9, 10, 11, 12
ST_HDR = 16


def status_ints(n: int) -> int:
    return ST_HDR + 4 * n


class VsConfig(C.Structure):
    _fields_ = [("k", C.c_int32), ("n", C.c_int32), ("max_candidates", C.c_int32),
                ("max_len", C.c_int32), ("vocab_size", C.c_int32), ("sos", C.c_int32),
                ("eos", C.c_int32), ("policy", C.c_int32), ("capacity", C.c_int32),
                ("refill_threshold", C.c_int32), ("no_drain", C.c_int32), ("delta", C.c_double)]


_P = C.c_void_p
STATE_FIELDS = [
    "slot_input", "slot_lt", "slot_emitted", "slot_width", "slot_active", "slot_src_len",
    "slot_flags", "slot_seed", "c_score", "c_len", "c_row", "c_fin", "c_hash", "hist", "live",
    "counters", "sel", "sel_off", "row_slot", "row_cand", "row_phys", "row_len", "src_off",
    "src_tok", "out_count", "out_len", "out_score", "out_tok", "top_tok", "top_logp", "row_lse",
    "copy_list", "n_copy", "status", "c_act", "top_logp64", "out_off",
]


class VsState(C.Structure):
    _fields_ = [(f, _P) for f in STATE_FIELDS]


class VsHashParams(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("scale", C.c_float), ("eos_bias", C.c_float),
                ("power", C.c_int32), ("dtype", C.c_int32)]


# Every symbol include/varstream.h declares (checked by tests/test_native_exports.py).
EXPORTS = ("vs_version", "vs_row_lse_topm", "vs_row_lse_topm_ws", "vs_row_lse_topm_ws_bytes", "vs_beam_step",
           "vs_beam_step_schedule", "vs_schedule", "vs_schedule_mirror", "vs_rows_copy",
           "vs_scatter_rows", "vs_hash_encode", "vs_hash_logits", "vs_row_attention", "vs_row_attention_grouped",
           "vs_proj_lse_topm", "vs_proj_lse_topm_ws_bytes", "vs_row_topm_f64", "vs_layer_norm_bf16")

_lib = None


def load_library(path: Path | None = None) -> C.CDLL:
    """Load libvarstream.so (raises if absent — there is no fallback)."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = Path(path or os.environ.get("VARSTREAM_LIB", LIB_PATH))
    if not p.exists():
        raise RuntimeError(f"varstream CUDA library not built: {p} (run __graft_entry__.build())")
    lib = C.CDLL(str(p))
    i32, i64, u64, vp = C.c_int32, C.c_int64, C.c_uint64, C.c_void_p
    sig = {
        "vs_version": ([], i32),
        "vs_row_lse_topm": ([vp, i32, i64, i32, i32, i32, vp, i32, vp, vp, vp, vp, vp], i32),
        "vs_row_lse_topm_ws": ([vp, i32, i64, i32, i32, i32, vp, i32, vp, vp, vp, vp, vp, C.c_size_t, vp],
                               i32),
        "vs_row_lse_topm_ws_bytes": ([i32, i32, i32], C.c_size_t),
        "vs_row_topm_f64": ([vp, i64, i32, i32, i32, vp, i32, vp, vp, vp, vp], i32),
        "vs_layer_norm_bf16": ([vp, i64, vp, i64, i32, i32, C.c_float, vp], i32),
        "vs_beam_step": ([C.POINTER(VsConfig), C.POINTER(VsState), i32, vp], i32),
        "vs_schedule": ([C.POINTER(VsConfig), C.POINTER(VsState), i32, i32, i32, i32, i32, vp], i32),
        "vs_schedule_mirror": ([C.POINTER(VsConfig), C.POINTER(VsState), i32, i32, i32, i32, i32, vp, vp], i32),
        "vs_beam_step_schedule": ([C.POINTER(VsConfig), C.POINTER(VsState), i32, i32, i32, i32, vp, vp], i32),
        "vs_rows_copy": ([vp, i64, i32, i64, i64, vp, vp, i32, vp], i32),
        "vs_scatter_rows": ([vp, i64, vp, i64, i64, vp, vp, i32, vp], i32),
        "vs_hash_encode": ([C.POINTER(VsConfig), C.POINTER(VsState), u64, vp], i32),
        "vs_proj_lse_topm": ([vp, i64, vp, i64, i32, vp, i32, i32, i32, i32, i32, vp, vp, i64, vp, vp, vp, vp,
                              vp, C.c_size_t, vp], i32),
        "vs_proj_lse_topm_ws_bytes": ([i32, i32], C.c_size_t),
        "vs_row_attention": ([vp, i64, vp, vp, i64, i64, vp, vp, vp, vp, i64, vp, i64, i32, i32, C.c_float,
                              i32, vp, i32, vp], i32),
        "vs_row_attention_grouped": ([vp, i64, vp, vp, i64, i64, vp, vp, vp, vp, i32, vp, i64, i32, i32,
                                      C.c_float, vp], i32),
        "vs_hash_logits": ([C.POINTER(VsConfig), C.POINTER(VsState), C.POINTER(VsHashParams), vp,
                            i64, i32, vp], i32),
    }
    for name, (args, ret) in sig.items():
        fn = getattr(lib, name)
        fn.argtypes, fn.restype = args, ret
    if path is None:
        _lib = lib
    return lib


_vsmat = None


def load_vsmat():
    """The host-runtime extension (_lib/_vsmat*.so, built by __graft_entry__.build())
    that materialises decode outputs as Candidate lists in bulk."""
    global _vsmat
    if _vsmat is None:
        import importlib.machinery
        import importlib.util
        import sysconfig

        p = LIB_PATH.parent / ("_vsmat" + sysconfig.get_config_var("EXT_SUFFIX"))
        if not p.exists():
            raise RuntimeError(f"host extension not built: {p} (run __graft_entry__.build())")
        loader = importlib.machinery.ExtensionFileLoader("_vsmat", str(p))
        spec = importlib.util.spec_from_loader("_vsmat", loader)
        mod = importlib.util.module_from_spec(spec)
        loader.exec_module(mod)
        _vsmat = mod
    return _vsmat


def check(rc: int, what: str) -> None:
    """Map a C-ABI status onto the reference taxonomy (bb/errors.py)."""
    if rc == VS_OK:
        return
    if rc == VS_ERR_CONFIG:
        raise ConfigError(f"{what}: invalid configuration or arguments")
    if rc == VS_ERR_INVARIANT:
        raise InvariantViolation(f"{what}: device contract violated")
    raise RuntimeError(f"{what}: CUDA error (code {rc})")
