"""ctypes loader for libmcapq.so (the C ABI in include/mcapq.h).

Argument marshalling only.  If the library is missing this raises: there is no
CPU or PyTorch fallback anywhere in this package.
"""
from __future__ import annotations

import ctypes
import os
from pathlib import Path

_PKG = Path(__file__).resolve().parent
# MCAPQ_LIB: diagnostic A/B runs only (another build of the same sources, e.g. under _ab/)
LIB_PATH = Path(os.environ.get("MCAPQ_LIB") or (_PKG / "lib" / "libmcapq.so"))

P = ctypes.c_void_p
I64 = ctypes.c_int64
I32 = ctypes.c_int
SZ = ctypes.c_size_t
DBL = ctypes.c_double

# name -> (restype, argtypes); mirrors include/mcapq.h one for one
SIGNATURES = {
    "mcapq_abi_version": (I32, []),
    "mcapq_last_error": (ctypes.c_char_p, []),
    "mcapq_status_string": (ctypes.c_char_p, [I32]),
    "mcapq_device_sms": (I32, []),
    "mcapq_set_pdl": (I32, [I32]),
    "mcapq_debug_stream_trace": (SZ, [P, SZ]),
    "mcapq_debug_read_bw": (I32, [P, SZ, P, P]),
    "mcapq_debug_linear_peers": (I32, [I32, P, P, I64, I64, P, P, I32, P, I32, P]),
    "mcapq_w4_nib_bytes": (SZ, [I64, I64]),
    "mcapq_w4_scale_bytes": (SZ, [I64, I64]),
    "mcapq_pack_w4": (I32, [P, I32, I64, I64, I64, P, P, P, P]),
    "mcapq_quant_a8": (I32, [P, I64, I64, I64, P, P, P, P]),
    "mcapq_w4a8": (I32, [P, P, I64, I64, P, P, P, I64, P, I32, I64, P]),
    "mcapq_workspace_bytes": (SZ, [I32, I64, I64, I64]),
    "mcapq_w4a8_x": (I32, [P, P, I64, I64, P, I64, I64, P, I32, I64, P, SZ, P]),
    "mcapq_w4a16": (I32, [P, P, I64, I64, P, I64, I64, P, I32, I64, P]),
    "mcapq_w4a16_bf16deq": (I32, [P, P, I64, I64, P, I64, I64, P, I32, I64, P]),
    "mcapq_prefill_workspace_bytes": (SZ, [I64, I64]),
    "mcapq_dequant_w4_bf16": (I32, [P, P, I64, I64, P, P]),
    "mcapq_bf16w_gemm": (I32, [P, I64, I64, P, I64, I64, P, I32, I64, P]),
    "mcapq_w4a16_bf16deq_prefill": (I32, [P, P, I64, I64, P, I64, I64, P, I32, I64, P, SZ, P]),
    "mcapq_argmax_workspace_bytes": (SZ, [I32, I64, I64, I64, I32]),
    "mcapq_linear_argmax": (I32, [I32, P, P, I64, I64, P, I64, I64, P, P, P, SZ, P]),
    "mcapq_argmax_keys": (I32, [I32, P, P, I64, I64, P, I64, I64, I64, P, P, SZ, P]),
    "mcapq_argmax_combine": (I32, [P, I32, I64, P, P, P]),
    "mcapq_linear": (I32, [I32, P, P, I64, I64, P, I64, I64, P, I32, I64, P, SZ, P]),
    "mcapq_linear_group": (I32, [I32, I32, P, P, P, I64, P, I64, I64, P, I32, P, P, SZ, P]),
    "mcapq_host_workspace_bytes": (SZ, [I32, I64, I64, I64]),
    "mcapq_linear_host": (I32, [I32, P, P, I64, I64, P, I64, P, I32, P, SZ, P]),
    "mcapq_w4a8_group_dots": (I32, [P, I64, I64, P, P, I64, P, I32, P]),
    "mcapq_debug_stream_dump_workspace_bytes": (SZ, [I64]),
    "mcapq_debug_stream_w4a8_dump": (I32, [P, P, I64, I64, P, P, P, P, P, P, SZ, P]),
    "mcapq_profile_parse": (I32, [ctypes.c_char_p, SZ, DBL, ctypes.POINTER(P)]),
    "mcapq_profile_layers": (I32, [P]),
    "mcapq_profile_tau": (DBL, [P]),
    "mcapq_profile_scores": (I32, [P, P, I32]),
    "mcapq_profile_routes": (I32, [P, P, I32]),
    "mcapq_profile_free": (None, [P]),
    "mcapq_profile_write_json": (I32, [P, I32, I32, DBL, ctypes.c_char_p, SZ, ctypes.POINTER(SZ)]),
    "mcapq_mcap_workspace_bytes": (SZ, [I64]),
    "mcapq_mcap_accumulate": (I32, [P, I64, I64, P, I64, I64, P, I64, I64, I64, DBL, P, P, SZ, P]),
    "mcapq_stack_create": (I32, [I32, P, I64, ctypes.POINTER(P)]),
    "mcapq_stack_set": (I32, [P, I32, I32, I32, P, P, I64, I64, P, P, I32]),
    "mcapq_stack_run": (I32, [P, I64, P]),
    "mcapq_stack_capture": (I32, [P, I64, P]),
    "mcapq_stack_replay": (I32, [P, P]),
    "mcapq_stack_weight_bytes": (SZ, [P]),
    "mcapq_stack_launches": (I32, [P, I64]),
    "mcapq_stack_host_bytes": (SZ, [P, I64, I32]),
    "mcapq_stack_step_host": (I32, [P, I64, P, P, P]),
    "mcapq_stack_destroy": (None, [P]),
    "mcapq_comm_unique_id": (I32, [P]),
    "mcapq_comm_init": (I32, [P, I32, I32, ctypes.POINTER(P)]),
    "mcapq_comm_world": (I32, [P]),
    "mcapq_comm_rank": (I32, [P]),
    "mcapq_colshard_workspace_bytes": (SZ, [I32, I64, I64, I64, I32]),
    "mcapq_linear_colshard": (I32, [P, I32, P, P, I64, I64, P, I64, P, I32, P, SZ, I32, P]),
    "mcapq_comm_window_alloc": (I32, [P, SZ, P]),
    "mcapq_comm_window_free": (I32, [P, P]),
    "mcapq_colshard_assemble": (I32, [P, P, I64, I64, I32, I32, P]),
    "mcapq_linear_colshard_argmax": (I32, [P, I32, P, P, I64, I64, P, I64, P, P, P, SZ, P]),
    "mcapq_rowshard_workspace_bytes": (SZ, [I32, I64, I64, I64, I32]),
    "mcapq_linear_rowshard": (I32, [P, I32, P, P, I64, I64, P, I64, I64, P, I32, P, SZ, I32, P]),
    "mcapq_rowshard_reduce": (I32, [P, I32, I64, I64, P, I32, P]),
    "mcapq_comm_destroy": (None, [P]),
}


class McapqError(RuntimeError):
    def __init__(self, status: int, fn: str, msg: str):
        super().__init__(f"{fn} -> status {status}: {msg}")
        self.status = status


_lib = None


def load(path: str | os.PathLike | None = None) -> ctypes.CDLL:
    """Load libmcapq.so (build it first with paper_2604_21026_b200.build)."""
    global _lib
    if _lib is not None:
        return _lib
    p = Path(path) if path else LIB_PATH
    if not p.exists():
        raise ImportError(f"{p} is missing: run `python -m paper_2604_21026_b200.build` (no fallback path exists)")
    L = ctypes.CDLL(str(p))
    for name, (res, args) in SIGNATURES.items():
        if name.startswith("mcapq_debug_") and os.environ.get("MCAPQ_LIB") and not hasattr(L, name):
            continue   # an older build under A/B (MCAPQ_LIB) may predate a diagnostic entry
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return _lib


def check(status: int, fn: str):
    if status != 0:
        msg = load().mcapq_last_error().decode(errors="replace")
        raise McapqError(status, fn, msg)
