"""CPU oracle for the MCAP/NVE mixed-precision decode linear (arXiv 2604.21026).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product (``paper_2604_21026_b200``) never imports it, and the two
share no code: the arithmetic lives in ``oracle/mcapq_oracle.c`` (plain C, no
CUDA headers) and in the small pure-Python functions below.

Each function cites the passage it follows (``P:n`` = PAPER.md line, ``S:n`` =
SPEC.md line) and the DESIGN.md reading label (A1..A22, T).  Pins: see
``tests/test_oracle_*.py`` and DESIGN.md "Oracle pins".  Parity status per
function is listed in DESIGN.md; no function here is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import json
import math
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_SRC = _HERE / "mcapq_oracle.c"
_LIB = _HERE / "_build" / "libmcapq_oracle.so"

W4A8, W4A16 = 0, 1
TAU_DEFAULT = 0.7
EPS_DEFAULT = 1e-9         # reading A14; the paper gives no value


def build(force: bool = False) -> Path:
    """Compile the C oracle (gcc, IEEE fp32, no contraction, OpenMP over rows)."""
    if _LIB.exists() and not force and _LIB.stat().st_mtime >= _SRC.stat().st_mtime:
        return _LIB
    _LIB.parent.mkdir(parents=True, exist_ok=True)
    tmp = _LIB.with_suffix(f".{os.getpid()}.tmp")
    cmd = ["gcc", "-O2", "-std=c99", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
           "-shared", "-fPIC", str(_SRC), "-o", str(tmp), "-lm"]
    subprocess.run(cmd, check=True)
    os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(str(_LIB))
        P = ctypes.c_void_p
        I64 = ctypes.c_int64
        L.oracle_f32_to_f16.argtypes = [ctypes.c_float]
        L.oracle_f32_to_f16.restype = ctypes.c_uint16
        L.oracle_f16_to_f32.argtypes = [ctypes.c_uint16]
        L.oracle_f16_to_f32.restype = ctypes.c_float
        L.oracle_q4_0_block.argtypes = [P, P, P]
        L.oracle_pack_w4.argtypes = [P, I64, I64, P, P]
        L.oracle_dequant_w4.argtypes = [P, P, I64, I64, P]
        L.oracle_dequant_w4.restype = None
        L.oracle_export_q4_0_aos.argtypes = [P, P, I64, I64, P]
        L.oracle_export_q4_0_aos.restype = None
        L.oracle_quant_a8.argtypes = [P, I64, I64, P, P, P]
        L.oracle_w4a8_group_dots.argtypes = [P, I64, I64, P, P, I64, P]
        L.oracle_w4a8.argtypes = [P, P, I64, I64, P, P, P, I64, P, P]
        L.oracle_w4a16.argtypes = [P, P, I64, I64, P, I64, P, P]
        L.oracle_w4a16_bf16deq.argtypes = [P, P, I64, I64, P, I64, P, P]
        for f in ("oracle_f32_to_f16_array", "oracle_f16_to_f32_array", "oracle_f32_to_bf16_array"):
            getattr(L, f).argtypes = [P, I64, P]
            getattr(L, f).restype = None
        L.oracle_count_f16_mismatch.argtypes = [ctypes.c_uint32, ctypes.c_uint32, P]
        L.oracle_count_f16_mismatch.restype = ctypes.c_int64
        _lib = L
    return _lib


class OracleError(RuntimeError):
    pass


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float32))


def _check(status: int, what: str):
    if status == 1:
        raise OracleError(f"{what}: invalid shape (k % 32 != 0 or negative size)")
    if status == 3:
        raise OracleError(f"{what}: non-finite input or fp16 scale overflow (S:287, S:304, A4)")


# --------------------------------------------------------------------------
# IEEE conversions
# --------------------------------------------------------------------------
def f32_to_f16_bits(x) -> np.ndarray:
    x = _f32(x)
    out = np.empty(x.shape, np.uint16)
    lib().oracle_f32_to_f16_array(_p(x), x.size, _p(out))
    return out


def f16_bits_to_f32(h) -> np.ndarray:
    h = np.ascontiguousarray(np.asarray(h, dtype=np.uint16))
    out = np.empty(h.shape, np.float32)
    lib().oracle_f16_to_f32_array(_p(h), h.size, _p(out))
    return out


def f32_to_bf16_bits(x) -> np.ndarray:
    x = _f32(x)
    out = np.empty(x.shape, np.uint16)
    lib().oracle_f32_to_bf16_array(_p(x), x.size, _p(out))
    return out


def bf16_bits_to_f32(b) -> np.ndarray:
    """bf16 -> fp32 is exact: the bf16 bits are the top half of the fp32."""
    b = np.asarray(b, dtype=np.uint16)
    return (b.astype(np.uint32) << 16).view(np.float32)


# --------------------------------------------------------------------------
# a1: Q4_0 pack
# --------------------------------------------------------------------------
def pack_w4(w, check: bool = True):
    """W[n, k] (fp32 values) -> (nib uint8 [n, k/2], scale fp16 bits uint16 [n, k/32])."""
    w = _f32(w)
    n, k = w.shape
    nib = np.empty((n, k // 2), np.uint8)
    scale = np.empty((n, max(k // 32, 0)), np.uint16)
    st = lib().oracle_pack_w4(_p(w), n, k, _p(nib), _p(scale))
    if check:
        _check(st, "pack_w4")
    return nib, scale


def pack_w4_status(w):
    w = _f32(w)
    n, k = w.shape
    nib = np.empty((n, k // 2), np.uint8)
    scale = np.empty((n, k // 32), np.uint16)
    st = lib().oracle_pack_w4(_p(w), n, k, _p(nib), _p(scale))
    return st, nib, scale


def dequant_w4(nib, scale) -> np.ndarray:
    nib = np.ascontiguousarray(nib, np.uint8)
    scale = np.ascontiguousarray(scale, np.uint16)
    n, k = nib.shape[0], nib.shape[1] * 2
    w = np.empty((n, k), np.float32)
    lib().oracle_dequant_w4(_p(nib), _p(scale), n, k, _p(w))
    return w


def export_q4_0_aos(nib, scale) -> bytes:
    """18-byte Q4_0 blocks [d f16 LE][16 nibble bytes]."""
    nib = np.ascontiguousarray(nib, np.uint8)
    scale = np.ascontiguousarray(scale, np.uint16)
    n, k = nib.shape[0], nib.shape[1] * 2
    out = np.empty(n * (k // 32) * 18, np.uint8)
    lib().oracle_export_q4_0_aos(_p(nib), _p(scale), n, k, _p(out))
    return out.tobytes()


def codes(nib) -> np.ndarray:
    """Unsigned 4-bit codes c[n, k] from the split layout (byte t = c_t | c_{t+16} << 4)."""
    nib = np.asarray(nib, np.uint8)
    n, kh = nib.shape
    b = nib.reshape(n, kh // 16, 16)
    c = np.concatenate([b & 0x0F, b >> 4], axis=2)
    return c.reshape(n, kh * 2).astype(np.int32)


# --------------------------------------------------------------------------
# a2: activation quantisation
# --------------------------------------------------------------------------
def quant_a8(x, check: bool = True):
    """x[m, k] -> (q int8 [m, k], s fp32 [m, k/32], sq int32 [m, k/32])."""
    x = _f32(x)
    if x.ndim == 1:
        x = x[None, :]
    m, k = x.shape
    q = np.empty((m, k), np.int8)
    s = np.empty((m, k // 32), np.float32)
    sq = np.empty((m, k // 32), np.int32)
    st = lib().oracle_quant_a8(_p(x), m, k, _p(q), _p(s), _p(sq))
    if check:
        _check(st, "quant_a8")
    return q, s, sq


# --------------------------------------------------------------------------
# a3/a5: W4A8
# --------------------------------------------------------------------------
def w4a8_group_dots(nib, q, sq) -> np.ndarray:
    """D[m, n, G] = sumi - 8*sum_x per block, exact int32."""
    nib = np.ascontiguousarray(nib, np.uint8)
    q = np.ascontiguousarray(q, np.int8)
    sq = np.ascontiguousarray(sq, np.int32)
    n, k = nib.shape[0], nib.shape[1] * 2
    m = q.shape[0]
    D = np.empty((m, n, k // 32), np.int32)
    _check(lib().oracle_w4a8_group_dots(_p(nib), n, k, _p(q), _p(sq), m, _p(D)), "w4a8_group_dots")
    return D


def w4a8(nib, scale, q, s, sq):
    """-> (y32 [m, n] fp32 in increasing-g order, y64 [m, n] fp64 reference)."""
    nib = np.ascontiguousarray(nib, np.uint8)
    scale = np.ascontiguousarray(scale, np.uint16)
    q = np.ascontiguousarray(q, np.int8)
    s = np.ascontiguousarray(s, np.float32)
    sq = np.ascontiguousarray(sq, np.int32)
    n, k = nib.shape[0], nib.shape[1] * 2
    m = q.shape[0]
    y32 = np.empty((m, n), np.float32)
    y64 = np.empty((m, n), np.float64)
    _check(lib().oracle_w4a8(_p(nib), _p(scale), n, k, _p(q), _p(s), _p(sq), m, _p(y32), _p(y64)), "w4a8")
    return y32, y64


def w4a8_from_x(nib, scale, x):
    """Quantise then multiply: the W4A8 route's whole semantics for bf16 x."""
    q, s, sq = quant_a8(x)
    return w4a8(nib, scale, q, s, sq)


# --------------------------------------------------------------------------
# a4: W4A16 exact dequant; a6: bf16-dequant batched semantics (A13)
# --------------------------------------------------------------------------
def w4a16(nib, scale, x):
    nib = np.ascontiguousarray(nib, np.uint8)
    scale = np.ascontiguousarray(scale, np.uint16)
    x = _f32(x)
    if x.ndim == 1:
        x = x[None, :]
    n, k = nib.shape[0], nib.shape[1] * 2
    m = x.shape[0]
    y32 = np.empty((m, n), np.float32)
    y64 = np.empty((m, n), np.float64)
    _check(lib().oracle_w4a16(_p(nib), _p(scale), n, k, _p(x), m, _p(y32), _p(y64)), "w4a16")
    return y32, y64


def w4a16_bf16deq(nib, scale, x):
    nib = np.ascontiguousarray(nib, np.uint8)
    scale = np.ascontiguousarray(scale, np.uint16)
    x = _f32(x)
    if x.ndim == 1:
        x = x[None, :]
    n, k = nib.shape[0], nib.shape[1] * 2
    m = x.shape[0]
    y32 = np.empty((m, n), np.float32)
    y64 = np.empty((m, n), np.float64)
    _check(lib().oracle_w4a16_bf16deq(_p(nib), _p(scale), n, k, _p(x), m, _p(y32), _p(y64)), "w4a16_bf16deq")
    return y32, y64


# --------------------------------------------------------------------------
# NEXT-3: MCAP raw scores (Alg. 1 lines 1-10)
# --------------------------------------------------------------------------
def mcap_raw_scores(prompts):
    """Alg. 1 lines 1-10 written out.  prompts: k prompts, each a list over the L layers
    of (q, v, ffn) arrays [|p_j|, n] (the layer's Q x_t, V x_t and FFN(x_t) rows).
        a_attn = || [Q x_t, V x_t] ||_2          (line 5)
        a_ffn  = || FFN(x_t) ||_2                (line 6)
        s_i    = 1/k sum_j 1/|p_j| sum_t (a_attn + a_ffn)     (line 10)
    in fp64.  -> [s_1 .. s_L]."""
    k = len(prompts)
    L = len(prompts[0])
    s = [0.0] * L
    for layers in prompts:
        for i, (q, v, f) in enumerate(layers):
            q = np.asarray(q, np.float64)
            v = np.asarray(v, np.float64)
            f = np.asarray(f, np.float64)
            m = q.shape[0]
            total = 0.0
            for t in range(m):
                a_attn = math.sqrt(float(np.sum(q[t] * q[t])) + float(np.sum(v[t] * v[t])))
                a_ffn = math.sqrt(float(np.sum(f[t] * f[t])))
                total += a_attn + a_ffn
            s[i] += total / m / k
    return s


# --------------------------------------------------------------------------
# a7: profile -> routes (Alg. 1 lines 8-13; A14)
# --------------------------------------------------------------------------
def minmax_normalize(scores, eps: float = EPS_DEFAULT):
    """Alg. 1 lines 8-12: degenerate (max-min < eps) -> all 0."""
    s = [float(v) for v in scores]
    lo, hi = min(s), max(s)
    if hi - lo < eps:
        return [0.0 for _ in s]
    return [(v - lo) / (hi - lo) for v in s]


def route_layers(norm_scores, tau: float = TAU_DEFAULT):
    """route(i) = W4A16 iff s^_i >= tau else W4A8."""
    return [W4A16 if v >= tau else W4A8 for v in norm_scores]


def routes_from_profile(text: str, tau_override: float | None = None):
    """Profile JSON (SURVEY §8b schema) -> (normalised scores, tau, routes)."""
    obj = json.loads(text)
    if not isinstance(obj, dict):
        raise OracleError("profile: not a JSON object")
    eps = float(obj.get("epsilon", EPS_DEFAULT))
    scores = obj.get("scores", obj.get("normalized_scores"))
    if scores is None:
        raw = obj.get("raw_scores")
        if raw is None:
            raise OracleError("profile: no scores / normalized_scores / raw_scores array")
        scores = minmax_normalize(raw, eps)
    scores = [float(v) for v in scores]
    if any((not math.isfinite(v)) or v < 0.0 or v > 1.0 for v in scores):
        raise OracleError("profile: normalised score outside [0, 1]")
    nl = obj.get("num_layers", obj.get("layers"))
    if nl is not None and int(nl) != len(scores):
        raise OracleError("profile: num_layers does not match the score array")
    tau = float(obj.get("tau", obj.get("threshold", TAU_DEFAULT)))
    if tau_override is not None and not math.isnan(tau_override):
        tau = float(tau_override)
    return scores, tau, route_layers(scores, tau)


# --------------------------------------------------------------------------
# a8: column-sharded linear, emulated (reading A22): rank r owns rows
# [r*N/P, (r+1)*N/P); the all-gather concatenates rank-major.
# --------------------------------------------------------------------------
def colshard_rows(n: int, world: int, rank: int):
    if n % world:
        raise OracleError("colshard: N % P != 0")
    per = n // world
    return rank * per, (rank + 1) * per


def colshard_linear(route: int, nib, scale, x, world: int):
    """Run each shard on its own row slice, then concatenate (the all-gather)."""
    n = nib.shape[0]
    outs = []
    for r in range(world):
        a, b = colshard_rows(n, world, r)
        if route == W4A8:
            y32, _ = w4a8_from_x(nib[a:b], scale[a:b], x)
        else:
            y32, _ = w4a16(nib[a:b], scale[a:b], x)
        outs.append(y32)
    return np.concatenate(outs, axis=1)


# --------------------------------------------------------------------------
# NEXT-2: row-parallel (K-sharded) linear, the Megatron partner of the column shard
# (SURVEY 8(f) NEXT-2).  Rank r owns the K-slice [r K/P, (r+1) K/P) of W and x; K/P is
# a whole number of 32-groups, so every Q4_0 block and every per-token
# quantisation group lies in one rank.  Each rank's partial is the
# routed linear on its slice; the all-reduce is their sum.
# --------------------------------------------------------------------------
def rowshard_cols(k: int, world: int, rank: int):
    if k % world or (k // world) % 32:
        raise OracleError("rowshard: K/P must be a whole number of 32-groups")
    per = k // world
    return rank * per, (rank + 1) * per


def rowshard_linear(route: int, nib, scale, x, world: int):
    """-> (y32 [m, n]: the fp32 partials summed in rank order, y64 [m, n]: the fp64
    partials summed).  x: [m, k] values (bf16-representable)."""
    x = _f32(x)
    if x.ndim == 1:
        x = x[None, :]
    k = nib.shape[1] * 2
    y32 = y64 = None
    for r in range(world):
        a, b = rowshard_cols(k, world, r)
        nb, sb, xs = nib[:, a // 2:b // 2], scale[:, a // 32:b // 32], x[:, a:b]
        p32, p64 = w4a8_from_x(nb, sb, xs) if route == W4A8 else w4a16(nb, sb, xs)
        y32 = p32.copy() if y32 is None else (y32 + p32).astype(np.float32)
        y64 = p64.copy() if y64 is None else y64 + p64
    return y32, y64


# --------------------------------------------------------------------------
# NEXT-2: greedy decode ("decode uses greedy (argmax) sampling")
def argmax_first(y):
    """Per row of y: the index of the largest value, the FIRST such index on ties
    (a plain left-to-right scan with IEEE '>' -- so -0.0 == +0.0 ties too).  y: [n]
    or [m, n] float; returns an int64 array [m] (or a scalar for 1-D y)."""
    a = np.asarray(y)
    rows = a.reshape(1, -1) if a.ndim == 1 else a
    out = np.empty(rows.shape[0], dtype=np.int64)
    for i in range(rows.shape[0]):
        r = rows[i].tolist()
        best, bi = r[0], 0
        for j in range(1, len(r)):
            if r[j] > best:
                best, bi = r[j], j
        out[i] = bi
    return int(out[0]) if a.ndim == 1 else out


def colshard_argmax(y, world: int):
    """The sharded greedy decode: each of `world` contiguous row shards (A22) takes its
    local argmax_first, then the winner is the largest local maximum, the lowest rank on
    ties (== the first global index).  y: [m, n] logits."""
    a = np.asarray(y)
    m, n = a.shape
    out = np.empty(m, dtype=np.int64)
    for i in range(m):
        best_v, best_j = None, -1
        for r in range(world):
            lo, hi = colshard_rows(n, world, r)
            j = lo + argmax_first(a[i, lo:hi])
            if best_v is None or a[i, j] > best_v:
                best_v, best_j = a[i, j], j
        out[i] = best_j
    return out
