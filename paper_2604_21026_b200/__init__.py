"""B200-native MCAP/NVE mixed-precision decode linear (arXiv 2604.21026).

A thin binding over the C ABI (include/mcapq.h, libmcapq.so): the functions
below only marshal torch tensors (device memory, the current CUDA stream) into
pointers and sizes.  Every step of the hot path runs in the library's sm_100a
kernels; there is no CPU fallback (a missing library raises ImportError on
first use).

    route(i) = W4A16 if s^_i >= tau else W4A8
    W4A8   : Q4_0 int4 x per-token/per-32-group int8, int32 group dots
    W4A16  : Q4_0 int4 dequantised against bf16 activations
"""
from __future__ import annotations

import ctypes
import math

import torch

from . import _lib
from ._lib import McapqError, check, load

W4A8, W4A16 = 0, 1
BF16, F32 = 0, 1

__all__ = [
    "W4A8", "W4A16", "BF16", "F32", "McapqError", "load", "pack_w4", "quant_a8", "w4a8", "w4a8_x", "w4a16",
    "w4a16_bf16deq", "dequant_w4_bf16", "bf16w_gemm", "w4a16_bf16deq_prefill",
    "linear", "linear_group", "linear_host", "w4a8_group_dots", "workspace_bytes", "host_workspace_bytes", "Profile",
    "profile_parse", "profile_write_json", "mcap_accumulate", "Stack", "Comm", "linear_colshard", "PackedW4",
    "colshard_assemble", "stream_w4a8_dump", "linear_argmax", "argmax_keys", "argmax_combine",
    "argmax_workspace_bytes", "linear_colshard_argmax", "linear_rowshard", "rowshard_reduce",
    "device_sms", "set_pdl", "debug_read_bw", "debug_linear_peers",
]


def _ptr(t: torch.Tensor | None):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _dt(dtype) -> int:
    if dtype == torch.bfloat16:
        return BF16
    if dtype == torch.float32:
        return F32
    raise McapqError(2, "dtype", f"unsupported dtype {dtype}")


def _need_cuda(*ts):
    for t in ts:
        if t is not None and not t.is_cuda:
            raise McapqError(1, "binding", "tensor is not on a CUDA device (no CPU path exists)")


def _act(x: torch.Tensor, k: int, what: str = "x") -> torch.Tensor:
    """Activations as a [M, K] bf16 row-major view (the C ABI reads raw bf16 bits)."""
    _need_cuda(x)
    if x.dtype != torch.bfloat16:
        raise McapqError(2, "binding", f"{what} must be bfloat16, got {x.dtype}")
    x2 = x if x.dim() == 2 else x.view(1, -1)
    if x2.dim() != 2 or x2.shape[1] != k or x2.stride(1) != 1:
        raise McapqError(1, "binding", f"{what} must be a row-major [M, {k}] tensor, got shape "
                                       f"{tuple(x.shape)} strides {tuple(x.stride())}")
    return x2


def _scratch(nbytes: int, device, stream=None) -> torch.Tensor:
    """Library workspace allocated on the stream the call runs on, so the caching
    allocator cannot hand it to other work before that stream's kernels finish."""
    if stream is None:
        return torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device)
    with torch.cuda.stream(stream):
        return torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device)


def device_sms() -> int:
    return load().mcapq_device_sms()


class PackedW4:
    """A packed Q4_0 weight: nib uint8 [N, K/2] + scale (fp16 bits as int16) [N, K/32]."""

    __slots__ = ("nib", "scale", "n", "k")

    def __init__(self, nib: torch.Tensor, scale: torch.Tensor):
        self.nib, self.scale = nib, scale
        self.n, self.k = nib.shape[0], nib.shape[1] * 2

    def shard(self, world: int, rank: int) -> "PackedW4":
        per = self.n // world
        return PackedW4(self.nib[rank * per:(rank + 1) * per], self.scale[rank * per:(rank + 1) * per])

    def kshard(self, world: int, rank: int) -> "PackedW4":
        """NEXT-2 row-parallel shard: the K-slice [r K/P, (r+1) K/P) of every row (whole
        Q4_0 blocks: K/P % 32 == 0), copied to its own contiguous [N, K/(2P)] planes."""
        kp = self.k // world
        if self.k % world or kp % 32:
            raise McapqError(1, "binding", f"K={self.k} does not split into {world} whole-group slices")
        a = rank * kp
        return PackedW4(self.nib[:, a // 2:(a + kp) // 2].contiguous(),
                        self.scale[:, a // 32:(a + kp) // 32].contiguous())

    @property
    def nbytes(self) -> int:
        return self.nib.numel() + 2 * self.scale.numel()


def pack_w4(w: torch.Tensor, dev_err: torch.Tensor | None = None, stream=None) -> PackedW4:
    """a1: W [N, K] bf16/fp32 (CUDA) -> PackedW4.  dev_err: optional int32[1] flag word."""
    _need_cuda(w)
    assert w.dim() == 2 and w.stride(1) == 1
    n, k = w.shape
    nib = torch.empty((n, k // 2), dtype=torch.uint8, device=w.device)
    scale = torch.empty((n, k // 32), dtype=torch.int16, device=w.device)
    check(load().mcapq_pack_w4(_ptr(w), _dt(w.dtype), n, k, w.stride(0), _ptr(nib), _ptr(scale), _ptr(dev_err),
                               _stream(stream)), "mcapq_pack_w4")
    return PackedW4(nib, scale)


def quant_a8(x: torch.Tensor, stream=None, out=None):
    """a2: x [M, K] bf16 -> (q int8 [M, K], sx fp32 [M, K/32], sq int32 [M, K/32]);
    out: optional preallocated (q, sx, sq)."""
    x2 = _act(x, x.shape[-1])
    m, k = x2.shape
    if out is not None:
        q, sx, sq = out
    else:
        q = torch.empty((m, k), dtype=torch.int8, device=x.device)
        sx = torch.empty((m, k // 32), dtype=torch.float32, device=x.device)
        sq = torch.empty((m, k // 32), dtype=torch.int32, device=x.device)
    check(load().mcapq_quant_a8(_ptr(x2), m, k, x2.stride(0), _ptr(q), _ptr(sx), _ptr(sq), _stream(stream)),
          "mcapq_quant_a8")
    return q, sx, sq


def _out(m, n, dtype, device, out):
    if out is not None:
        return out
    return torch.empty((m, n), dtype=dtype, device=device)


def w4a8(w: PackedW4, q, sx, sq, out_dtype=torch.float32, out=None, stream=None):
    """a3/a5 on pre-quantised activations (q int8 [M, K], sx fp32 / sq int32 [M, K/32])."""
    _need_cuda(w.nib, q, sx, sq)
    m = q.shape[0]
    for t, dt, cols, name in ((q, torch.int8, w.k, "q"), (sx, torch.float32, w.k // 32, "sx"),
                              (sq, torch.int32, w.k // 32, "sq")):
        if t.dtype != dt or tuple(t.shape) != (m, cols) or not t.is_contiguous():
            raise McapqError(1, "binding", f"{name} must be a contiguous {dt} [{m}, {cols}] tensor")
    y = _out(m, w.n, out_dtype, q.device, out)
    check(load().mcapq_w4a8(_ptr(w.nib), _ptr(w.scale), w.n, w.k, _ptr(q), _ptr(sx), _ptr(sq), m, _ptr(y),
                            _dt(y.dtype), y.stride(0), _stream(stream)), "mcapq_w4a8")
    return y


def workspace_bytes(route: int, m: int, n: int, k: int) -> int:
    return load().mcapq_workspace_bytes(route, m, n, k)


def host_workspace_bytes(route: int, m: int, n: int, k: int) -> int:
    return load().mcapq_host_workspace_bytes(route, m, n, k)


def _ws(route, m, n, k, device, ws, stream=None):
    if ws is not None:
        return ws
    return _scratch(workspace_bytes(route, m, n, k), device, stream)


def w4a8_x(w: PackedW4, x: torch.Tensor, out_dtype=torch.float32, out=None, ws=None, stream=None):
    """a2+a3/a5: quantise x then W4A8 (two PDL-chained launches)."""
    _need_cuda(w.nib)
    x2 = _act(x, w.k)
    m = x2.shape[0]
    y = _out(m, w.n, out_dtype, x.device, out)
    ws = _ws(W4A8, m, w.n, w.k, x.device, ws, stream)
    check(load().mcapq_w4a8_x(_ptr(w.nib), _ptr(w.scale), w.n, w.k, _ptr(x2), m, x2.stride(0), _ptr(y),
                              _dt(y.dtype), y.stride(0), _ptr(ws), ws.numel(), _stream(stream)), "mcapq_w4a8_x")
    return y


def w4a16(w: PackedW4, x: torch.Tensor, out_dtype=torch.float32, out=None, stream=None):
    """a4/a6: exact-dequant W4A16 on bf16 tensor cores."""
    _need_cuda(w.nib)
    x2 = _act(x, w.k)
    m = x2.shape[0]
    y = _out(m, w.n, out_dtype, x.device, out)
    check(load().mcapq_w4a16(_ptr(w.nib), _ptr(w.scale), w.n, w.k, _ptr(x2), m, x2.stride(0), _ptr(y),
                             _dt(y.dtype), y.stride(0), _stream(stream)), "mcapq_w4a16")
    return y


def w4a16_bf16deq(w: PackedW4, x: torch.Tensor, out_dtype=torch.float32, out=None, stream=None):
    """a6, bf16-dequant semantics: W^ = bf16(d (c - 8)), y = x W^T on tcgen05 (K % 256 == 0)."""
    _need_cuda(w.nib)
    x2 = _act(x, w.k)
    m = x2.shape[0]
    y = _out(m, w.n, out_dtype, x.device, out)
    check(load().mcapq_w4a16_bf16deq(_ptr(w.nib), _ptr(w.scale), w.n, w.k, _ptr(x2), m, x2.stride(0), _ptr(y),
                                     _dt(y.dtype), y.stride(0), _stream(stream)), "mcapq_w4a16_bf16deq")
    return y


def dequant_w4_bf16(w: PackedW4, out=None, stream=None) -> torch.Tensor:
    """NEXT-4: W^ = bf16_rne(d (c - 8)) as a bf16 [N, K] tensor (mcapq_dequant_w4_bf16)."""
    _need_cuda(w.nib)
    y = out if out is not None else torch.empty((w.n, w.k), dtype=torch.bfloat16, device=w.nib.device)
    check(load().mcapq_dequant_w4_bf16(_ptr(w.nib), _ptr(w.scale), w.n, w.k, _ptr(y), _stream(stream)),
          "mcapq_dequant_w4_bf16")
    return y


def bf16w_gemm(wdq: torch.Tensor, x: torch.Tensor, out_dtype=torch.float32, out=None, stream=None):
    """NEXT-4: y = x W^T for a resident bf16 W^ [N, K] on tcgen05 (mcapq_bf16w_gemm)."""
    _need_cuda(wdq)
    n, k = wdq.shape
    x2 = _act(x, k)
    m = x2.shape[0]
    y = _out(m, n, out_dtype, x.device, out)
    check(load().mcapq_bf16w_gemm(_ptr(wdq), n, k, _ptr(x2), m, x2.stride(0), _ptr(y), _dt(y.dtype), y.stride(0),
                                  _stream(stream)), "mcapq_bf16w_gemm")
    return y


def w4a16_bf16deq_prefill(w: PackedW4, x: torch.Tensor, out_dtype=torch.float32, out=None, ws=None, stream=None):
    """NEXT-4: dequantise once into ws, then the tcgen05 GEMM (mcapq_w4a16_bf16deq_prefill)."""
    _need_cuda(w.nib)
    x2 = _act(x, w.k)
    m = x2.shape[0]
    y = _out(m, w.n, out_dtype, x.device, out)
    if ws is None:
        ws = _scratch(load().mcapq_prefill_workspace_bytes(w.n, w.k), x.device, stream)
    check(load().mcapq_w4a16_bf16deq_prefill(_ptr(w.nib), _ptr(w.scale), w.n, w.k, _ptr(x2), m, x2.stride(0),
                                             _ptr(y), _dt(y.dtype), y.stride(0), _ptr(ws), ws.numel(),
                                             _stream(stream)), "mcapq_w4a16_bf16deq_prefill")
    return y


def set_pdl(enable: bool) -> bool:
    """Launch this thread's subsequent linears with programmatic dependent launch
    (mcapq_set_pdl); returns the previous setting."""
    return bool(load().mcapq_set_pdl(1 if enable else 0))


def linear(route: int, w: PackedW4, x: torch.Tensor, out_dtype=torch.float32, out=None, ws=None, stream=None):
    """Routed linear (a3-a6 by route)."""
    _need_cuda(w.nib)
    x2 = _act(x, w.k)
    m = x2.shape[0]
    y = _out(m, w.n, out_dtype, x.device, out)
    ws = _ws(route, m, w.n, w.k, x.device, ws, stream)
    check(load().mcapq_linear(route, _ptr(w.nib), _ptr(w.scale), w.n, w.k, _ptr(x2), m, x2.stride(0), _ptr(y),
                              _dt(y.dtype), y.stride(0), _ptr(ws), ws.numel(), _stream(stream)), "mcapq_linear")
    return y


def argmax_workspace_bytes(route: int, m: int, n: int, k: int, parts: int = 1) -> int:
    return load().mcapq_argmax_workspace_bytes(route, m, n, k, parts)


def linear_argmax(route: int, w: PackedW4, x: torch.Tensor, ws=None, stream=None):
    """NEXT-2 greedy decode: (idx int64 [M], val fp32 [M]) = argmax over the N outputs of the
    routed linear's fp32 logits, ties -> lowest index (mcapq_linear_argmax)."""
    _need_cuda(w.nib)
    x2 = _act(x, w.k)
    m = x2.shape[0]
    idx = torch.empty(m, dtype=torch.int64, device=x.device)
    val = torch.empty(m, dtype=torch.float32, device=x.device)
    ws = ws if ws is not None else _scratch(argmax_workspace_bytes(route, m, w.n, w.k), x.device, stream)
    check(load().mcapq_linear_argmax(route, _ptr(w.nib), _ptr(w.scale), w.n, w.k, _ptr(x2), m, x2.stride(0), _ptr(idx),
                                     _ptr(val), _ptr(ws), ws.numel(), _stream(stream)), "mcapq_linear_argmax")
    return idx, val


def argmax_keys(route: int, w: PackedW4, x: torch.Tensor, row_offset: int = 0, out=None, ws=None, stream=None):
    """NEXT-2 building block: per-token 64-bit argmax keys (as int64 bits) of this (shard of
    the) weight, global row index = row_offset + n (mcapq_argmax_keys)."""
    _need_cuda(w.nib)
    x2 = _act(x, w.k)
    m = x2.shape[0]
    keys = out if out is not None else torch.empty(m, dtype=torch.int64, device=x.device)
    ws = ws if ws is not None else _scratch(argmax_workspace_bytes(route, m, w.n, w.k), x.device, stream)
    check(load().mcapq_argmax_keys(route, _ptr(w.nib), _ptr(w.scale), w.n, w.k, _ptr(x2), m, x2.stride(0),
                                   int(row_offset), _ptr(keys), _ptr(ws), ws.numel(), _stream(stream)),
          "mcapq_argmax_keys")
    return keys


def argmax_combine(keys: torch.Tensor, stream=None):
    """(idx, val) of the largest key over the parts: keys int64 [P, M] (mcapq_argmax_combine)."""
    _need_cuda(keys)
    k2 = keys if keys.dim() == 2 else keys.view(1, -1)
    assert k2.dtype == torch.int64 and k2.is_contiguous()
    parts, m = k2.shape
    idx = torch.empty(m, dtype=torch.int64, device=keys.device)
    val = torch.empty(m, dtype=torch.float32, device=keys.device)
    check(load().mcapq_argmax_combine(_ptr(k2), parts, m, _ptr(idx), _ptr(val), _stream(stream)),
          "mcapq_argmax_combine")
    return idx, val


def linear_group(route: int, ws_list, x: torch.Tensor, out_dtype=torch.float32, outs=None, ws=None, stream=None):
    """Grouped routed linear: several PackedW4 sharing the same input x in one launch."""
    ws_list = list(ws_list)
    k = ws_list[0].k
    if any(w.k != k for w in ws_list):
        raise McapqError(1, "binding", "linear_group: every weight must have the same K")
    x2 = _act(x, k)
    m = x2.shape[0]
    cnt = len(ws_list)
    outs = outs if outs is not None else [torch.empty((m, w.n), dtype=out_dtype, device=x.device) for w in ws_list]
    arr = lambda T, vals: (T * cnt)(*vals)  # noqa: E731
    nibs = arr(ctypes.c_void_p, [w.nib.data_ptr() for w in ws_list])
    scs = arr(ctypes.c_void_p, [w.scale.data_ptr() for w in ws_list])
    ns = arr(ctypes.c_int64, [w.n for w in ws_list])
    ys = arr(ctypes.c_void_p, [y.data_ptr() for y in outs])
    lds = arr(ctypes.c_int64, [y.stride(0) for y in outs])
    ws = _ws(route, m, max(w.n for w in ws_list), k, x.device, ws, stream)
    check(load().mcapq_linear_group(route, cnt, ctypes.cast(nibs, ctypes.c_void_p), ctypes.cast(scs, ctypes.c_void_p),
                                    ctypes.cast(ns, ctypes.c_void_p), k, _ptr(x2), m, x2.stride(0),
                                    ctypes.cast(ys, ctypes.c_void_p), _dt(outs[0].dtype),
                                    ctypes.cast(lds, ctypes.c_void_p), _ptr(ws), ws.numel(), _stream(stream)),
          "mcapq_linear_group")
    return outs


def linear_host(route: int, w: PackedW4, x_host: torch.Tensor, y_host: torch.Tensor, ws: torch.Tensor,
                stream=None):
    """End-to-end routed linear from pinned host x into pinned host y (asynchronous)."""
    m, k = x_host.shape
    check(load().mcapq_linear_host(route, _ptr(w.nib), _ptr(w.scale), w.n, w.k, _ptr(x_host), m, _ptr(y_host),
                                   _dt(y_host.dtype), _ptr(ws), ws.numel(), _stream(stream)), "mcapq_linear_host")
    return y_host


def w4a8_group_dots(w: PackedW4, q, sq, mode: int = 1, stream=None):
    """Test entry: exact int32 D [M, N, K/32] through the dp4a (0) or IMMA (1) code."""
    m = q.shape[0]
    D = torch.empty((m, w.n, w.k // 32), dtype=torch.int32, device=q.device)
    check(load().mcapq_w4a8_group_dots(_ptr(w.nib), w.n, w.k, _ptr(q), _ptr(sq), m, _ptr(D), mode,
                                       _stream(stream)), "mcapq_w4a8_group_dots")
    return D


def stream_w4a8_dump(w: PackedW4, x: torch.Tensor, stream=None):
    """Test entry: the stream kernel's fused quantiser output (q, sx, sq) for one token
    and every block's exact D [N, K/32] (mcapq_debug_stream_w4a8_dump)."""
    _need_cuda(w.nib)
    x2 = _act(x, w.k)
    assert x2.shape[0] == 1
    dev = x.device
    q = torch.empty(w.k, dtype=torch.int8, device=dev)
    sx = torch.empty(w.k // 32, dtype=torch.float32, device=dev)
    sq = torch.empty(w.k // 32, dtype=torch.int32, device=dev)
    D = torch.empty((w.n, w.k // 32), dtype=torch.int32, device=dev)
    ws = _scratch(load().mcapq_debug_stream_dump_workspace_bytes(w.k), dev, stream)
    check(load().mcapq_debug_stream_w4a8_dump(_ptr(w.nib), _ptr(w.scale), w.n, w.k, _ptr(x2), _ptr(q), _ptr(sx),
                                              _ptr(sq), _ptr(D), _ptr(ws), ws.numel(), _stream(stream)),
          "mcapq_debug_stream_w4a8_dump")
    return q, sx, sq, D


# ------------------------------------------------------------------ profile
def debug_read_bw(buf: torch.Tensor, sink: torch.Tensor, stream=None):
    """Diagnostic: one streaming read of buf (the pure-read HBM ceiling; mcapq_debug_read_bw)."""
    _need_cuda(buf, sink)
    check(load().mcapq_debug_read_bw(_ptr(buf), buf.numel() * buf.element_size(), _ptr(sink), _stream(stream)),
          "mcapq_debug_read_bw")


class Profile:
    """Dispatch table parsed by the library (a7)."""

    def __init__(self, handle):
        self._h = handle

    def __del__(self):
        if getattr(self, "_h", None):
            load().mcapq_profile_free(self._h)
            self._h = None

    @property
    def layers(self) -> int:
        return load().mcapq_profile_layers(self._h)

    @property
    def tau(self) -> float:
        return load().mcapq_profile_tau(self._h)

    def scores(self):
        n = self.layers
        buf = (ctypes.c_double * n)()
        check(load().mcapq_profile_scores(self._h, ctypes.cast(buf, ctypes.c_void_p), n), "mcapq_profile_scores")
        return list(buf)

    def routes(self):
        n = self.layers
        buf = (ctypes.c_uint8 * n)()
        check(load().mcapq_profile_routes(self._h, ctypes.cast(buf, ctypes.c_void_p), n), "mcapq_profile_routes")
        return list(buf)


def profile_parse(text: str | bytes, tau: float | None = None) -> Profile:
    b = text.encode() if isinstance(text, str) else bytes(text)
    h = ctypes.c_void_p()
    check(load().mcapq_profile_parse(b, len(b), float("nan") if tau is None else float(tau), ctypes.byref(h)),
          "mcapq_profile_parse")
    return Profile(h)


def profile_write_json(raw_scores, prompts: int, tau: float = 0.7) -> str:
    """NEXT-3: the profile artifact (JSON) from raw per-layer scores (mcapq_profile_write_json)."""
    L = len(raw_scores)
    arr = (ctypes.c_double * L)(*[float(v) for v in raw_scores])
    n = ctypes.c_size_t(0)
    cap = 64 + 32 * L
    buf = ctypes.create_string_buffer(cap)
    check(load().mcapq_profile_write_json(ctypes.cast(arr, ctypes.c_void_p), L, int(prompts), float(tau), buf, cap,
                                          ctypes.byref(n)), "mcapq_profile_write_json")
    return buf.value.decode()


def mcap_accumulate(yq: torch.Tensor, yv: torch.Tensor, yffn: torch.Tensor, weight: float, score: torch.Tensor,
                    ws: torch.Tensor | None = None, stream=None):
    """NEXT-3 (Alg. 1 lines 3-10): score (fp64 device scalar) += weight * sum_t (||[q_t, v_t]|| + ||ffn_t||)
    over the m token rows of one layer's bf16 linear outputs."""
    _need_cuda(yq, yv, yffn, score)
    for t in (yq, yv, yffn):
        if t.dtype != torch.bfloat16 or t.dim() != 2 or t.stride(1) != 1:
            raise McapqError(1, "binding", "mcap_accumulate: bf16 [m, n] row-major tensors expected")
    if score.dtype != torch.float64:
        raise McapqError(2, "dtype", "score must be float64")
    m = yq.shape[0]
    if ws is None:
        ws = _scratch(load().mcapq_mcap_workspace_bytes(m), yq.device, stream)
    check(load().mcapq_mcap_accumulate(_ptr(yq), yq.stride(0), yq.shape[1], _ptr(yv), yv.stride(0), yv.shape[1],
                                       _ptr(yffn), yffn.stride(0), yffn.shape[1], m, float(weight), _ptr(score),
                                       _ptr(ws), ws.numel(), _stream(stream)), "mcapq_mcap_accumulate")
    return score


# ------------------------------------------------------------------ stack
class Stack:
    """Routed decode-linear stack (a9); the library owns its workspace and graph."""

    def __init__(self, routes, max_m: int = 1):
        self.routes = [int(r) for r in routes]
        buf = (ctypes.c_uint8 * len(self.routes))(*self.routes)
        h = ctypes.c_void_p()
        check(load().mcapq_stack_create(len(self.routes), ctypes.cast(buf, ctypes.c_void_p), max_m, ctypes.byref(h)),
              "mcapq_stack_create")
        self._h = h
        self._keep = []

    def __del__(self):
        if getattr(self, "_h", None):
            load().mcapq_stack_destroy(self._h)
            self._h = None

    def set(self, layer: int, slot: int, input_id: int, w: PackedW4, x: torch.Tensor, y: torch.Tensor):
        _act(x, w.k)
        if y.shape[-1] != w.n or y.stride(-1) != 1 or not y.is_contiguous():
            raise McapqError(1, "binding", f"y must be a contiguous [M, {w.n}] tensor")
        self._keep.append((w, x, y))
        check(load().mcapq_stack_set(self._h, layer, slot, input_id, _ptr(w.nib), _ptr(w.scale), w.n, w.k, _ptr(x),
                                     _ptr(y), _dt(y.dtype)), "mcapq_stack_set")

    def run(self, m: int = 1, stream=None):
        check(load().mcapq_stack_run(self._h, m, _stream(stream)), "mcapq_stack_run")

    def capture(self, m: int = 1, stream=None):
        check(load().mcapq_stack_capture(self._h, m, _stream(stream)), "mcapq_stack_capture")

    def replay(self, stream=None):
        check(load().mcapq_stack_replay(self._h, _stream(stream)), "mcapq_stack_replay")

    @property
    def weight_bytes(self) -> int:
        return load().mcapq_stack_weight_bytes(self._h)

    def launches(self, m: int = 1) -> int:
        return load().mcapq_stack_launches(self._h, m)

    def host_bytes(self, m: int = 1):
        """(input bytes, output bytes) of one end-to-end step."""
        return load().mcapq_stack_host_bytes(self._h, m, 0), load().mcapq_stack_host_bytes(self._h, m, 1)

    def step_host(self, x_host: torch.Tensor, y_host: torch.Tensor, m: int = 1, stream=None):
        """One end-to-end step: pinned host inputs -> graph replay -> pinned host outputs (async)."""
        bi, bo = self.host_bytes(m)
        assert x_host.numel() * x_host.element_size() >= bi and y_host.numel() * y_host.element_size() >= bo
        check(load().mcapq_stack_step_host(self._h, m, _ptr(x_host), _ptr(y_host), _stream(stream)),
              "mcapq_stack_step_host")


# ------------------------------------------------------------------ multi-GPU
class Comm:
    """Library-owned NCCL communicator; the unique id travels over a torch process group."""

    @staticmethod
    def bootstrap_id(group=None) -> bytes:
        """Rank 0 draws the NCCL unique id through the library; every rank of the
        torch process group receives the same 128 bytes."""
        import torch.distributed as dist
        obj = [None]
        if dist.get_rank(group) == 0:
            raw = (ctypes.c_uint8 * 128)()
            check(load().mcapq_comm_unique_id(ctypes.cast(raw, ctypes.c_void_p)), "mcapq_comm_unique_id")
            obj = [bytes(raw)]
        src = dist.get_global_rank(group, 0) if group is not None else 0
        dist.broadcast_object_list(obj, src=src, group=group)
        return obj[0]

    def __init__(self, group=None):
        import torch.distributed as dist
        world, rank = dist.get_world_size(group), dist.get_rank(group)
        raw = (ctypes.c_uint8 * 128)(*self.bootstrap_id(group))
        h = ctypes.c_void_p()
        check(load().mcapq_comm_init(ctypes.cast(raw, ctypes.c_void_p), world, rank, ctypes.byref(h)),
              "mcapq_comm_init")
        self._h, self.world, self.rank = h, world, rank

    def __del__(self):
        if getattr(self, "_h", None):
            load().mcapq_comm_destroy(self._h)
            self._h = None

    def workspace_bytes(self, route, m, n_full, k):
        return load().mcapq_colshard_workspace_bytes(route, m, n_full, k, self.world)

    def rowshard_workspace_bytes(self, route, m, n, k_shard):
        return load().mcapq_rowshard_workspace_bytes(route, m, n, k_shard, self.world)

    def window(self, n_full: int, dtype=torch.bfloat16, rows: int = 1) -> torch.Tensor:
        """COLLECTIVE: a [rows, n_full] buffer in an NCCL symmetric window
        (mcapq_comm_window_alloc): a y_full replica for linear_colshard(..., fused=True)
        (rows = 1), or the [P, n] fp32 partial slots of linear_rowshard(..., fused=True)
        (rows = P, dtype fp32); library-owned, released by free_window() or with the
        communicator."""
        es = torch.tensor([], dtype=dtype).element_size()
        ptr = ctypes.c_void_p()
        check(load().mcapq_comm_window_alloc(self._h, rows * n_full * es, ctypes.byref(ptr)),
              "mcapq_comm_window_alloc")

        class _Raw:   # a device pointer as a CUDA array (int16/int32 words, viewed as dtype below)
            __cuda_array_interface__ = {"shape": (rows, n_full), "typestr": "<i2" if es == 2 else "<i4",
                                        "data": (ptr.value, False), "version": 3}
        t = torch.as_tensor(_Raw(), device="cuda").view(dtype)
        self._windows = getattr(self, "_windows", []) + [(ptr.value, t)]
        return t

    def free_window(self, t: torch.Tensor):
        """COLLECTIVE: release a window from window()."""
        for i, (p, tt) in enumerate(getattr(self, "_windows", [])):
            if tt.data_ptr() == t.data_ptr():
                check(load().mcapq_comm_window_free(self._h, ctypes.c_void_p(p)), "mcapq_comm_window_free")
                del self._windows[i]
                return
        raise ValueError("not a window of this communicator")


def colshard_assemble(rank_major: torch.Tensor, world: int, out=None, stream=None) -> torch.Tensor:
    """a8 assembly: rank-major [P, M, N/P] -> y_full [M, N] (mcapq_colshard_assemble)."""
    _need_cuda(rank_major)
    P, m, per = rank_major.shape
    assert P == world and rank_major.is_contiguous()
    y = _out(m, P * per, rank_major.dtype, rank_major.device, out)
    check(load().mcapq_colshard_assemble(_ptr(rank_major), _ptr(y), m, P * per, world, _dt(y.dtype),
                                         _stream(stream)), "mcapq_colshard_assemble")
    return y


def linear_colshard_argmax(comm: Comm, route: int, w_shard: PackedW4, n_full: int, x: torch.Tensor, ws=None,
                           stream=None):
    """a8 + NEXT-2: column-sharded lm_head with a local argmax and a P x M key all-gather."""
    x2 = _act(x, w_shard.k)
    m = x2.shape[0]
    idx = torch.empty(m, dtype=torch.int64, device=x.device)
    val = torch.empty(m, dtype=torch.float32, device=x.device)
    ws = ws if ws is not None else _scratch(
        argmax_workspace_bytes(route, m, n_full // comm.world, w_shard.k, comm.world), x.device, stream)
    check(load().mcapq_linear_colshard_argmax(comm._h, route, _ptr(w_shard.nib), _ptr(w_shard.scale), n_full,
                                              w_shard.k, _ptr(x2), m, _ptr(idx), _ptr(val), _ptr(ws), ws.numel(),
                                              _stream(stream)), "mcapq_linear_colshard_argmax")
    return idx, val


def linear_colshard(comm: Comm, route: int, w_shard: PackedW4, n_full: int, x: torch.Tensor,
                    out_dtype=torch.bfloat16, out=None, ws=None, stream=None, fused: bool = False):
    """a8: column-sharded routed linear + NCCL all-gather into y_full [M, n_full].
    fused=True (M = 1): `out` must be a window tensor from Comm.window(); the GEMV epilogue
    stores straight into every rank's replica over NVLink, then one LSA barrier."""
    x2 = _act(x, w_shard.k)
    m = x2.shape[0]
    y = _out(m, n_full, out_dtype, x.device, out)
    ws = ws if ws is not None else _scratch(comm.workspace_bytes(route, m, n_full, w_shard.k), x.device, stream)
    check(load().mcapq_linear_colshard(comm._h, route, _ptr(w_shard.nib), _ptr(w_shard.scale), n_full, w_shard.k,
                                       _ptr(x2), m, _ptr(y), _dt(y.dtype), _ptr(ws), ws.numel(), int(bool(fused)),
                                       _stream(stream)),
          "mcapq_linear_colshard")
    return y


def linear_rowshard(comm: Comm, route: int, w_shard: PackedW4, x_shard: torch.Tensor, out_dtype=torch.bfloat16,
                    out=None, ws=None, stream=None, fused: bool = False):
    """NEXT-2: row-parallel (K-sharded) routed linear (mcapq_linear_rowshard): this rank's
    partial over its K-slice, summed over the ranks into y [M, n] on every rank (NCCL
    all-reduce; fused=True, M = 1: NVLink stores into every rank's window slots + LSA
    barriers + a rank-order sum -- `ws` must then be Comm.window(n, torch.float32, rows=P))."""
    x2 = _act(x_shard, w_shard.k)
    m = x2.shape[0]
    y = _out(m, w_shard.n, out_dtype, x_shard.device, out)
    if fused:
        assert ws is not None, "fused rowshard needs ws = Comm.window(n, torch.float32, rows=P)"
        wsb = ws.numel() * ws.element_size()
    else:
        ws = ws if ws is not None else _scratch(comm.rowshard_workspace_bytes(route, m, w_shard.n, w_shard.k),
                                                x_shard.device, stream)
        wsb = ws.numel() * ws.element_size()
    check(load().mcapq_linear_rowshard(comm._h, route, _ptr(w_shard.nib), _ptr(w_shard.scale), w_shard.n, w_shard.k,
                                       _ptr(x2), m, x2.stride(0), _ptr(y), _dt(y.dtype), _ptr(ws), wsb,
                                       int(bool(fused)), _stream(stream)), "mcapq_linear_rowshard")
    return y


def rowshard_reduce(partials: torch.Tensor, out_dtype=torch.bfloat16, out=None, stream=None) -> torch.Tensor:
    """NEXT-2 reduction / test entry: [P, M, N] fp32 partials -> y [M, N] = rank-order sum
    (mcapq_rowshard_reduce)."""
    _need_cuda(partials)
    assert partials.dtype == torch.float32 and partials.is_contiguous() and partials.dim() == 3
    P, m, n = partials.shape
    y = _out(m, n, out_dtype, partials.device, out)
    check(load().mcapq_rowshard_reduce(_ptr(partials), P, m, n, _ptr(y), _dt(y.dtype), _stream(stream)),
          "mcapq_rowshard_reduce")
    return y


def debug_linear_peers(route: int, w: PackedW4, x: torch.Tensor, y: torch.Tensor, peer_delta, stream=None):
    """Test entry: the fused epilogue's per-peer stores on one GPU (mcapq_debug_linear_peers):
    y (a view into one buffer) receives the rows, and so does every y + peer_delta[p] bytes."""
    x2 = _act(x, w.k)
    d = (ctypes.c_int64 * len(peer_delta))(*[int(v) for v in peer_delta])
    check(load().mcapq_debug_linear_peers(route, _ptr(w.nib), _ptr(w.scale), w.n, w.k, _ptr(x2), _ptr(y), _dt(y.dtype),
                                          ctypes.cast(d, ctypes.c_void_p), len(peer_delta), _stream(stream)),
          "mcapq_debug_linear_peers")
