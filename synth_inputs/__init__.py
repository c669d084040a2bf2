"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NO arithmetic of the method (no quantisation, no linear): it
only draws seeded bf16 weights and activations with the shapes and value
distributions of the paper's workloads (SURVEY §8(d)
D.1).  Both ``tests/`` and ``bench.py`` call it; ``oracle/`` and
``paper_2604_21026_b200/`` never import each other.

Shapes: Llama-3.2-1B / 3B and Llama-3.1-8B (public HF configs; the paper prints
only 14336x4096 at P:1432 and the layer counts at P:1346-1347).  Weights are
``nn.Linear.weight`` layout [N, K] (out, in).
"""
from __future__ import annotations

import torch

BASE_SEED = 260421026

# slot ids
SLOTS = ("q", "k", "v", "o", "gate", "up", "down", "lm_head")
SLOT_ID = {s: i for i, s in enumerate(SLOTS)}

MODELS = {
    #             L   hidden inter  q_out kv_out vocab
    "llama-3.2-1b": dict(layers=16, hidden=2048, inter=8192, q=2048, kv=512, vocab=128256),
    "llama-3.2-3b": dict(layers=28, hidden=3072, inter=8192, q=3072, kv=1024, vocab=128256),
    "llama-3.1-8b": dict(layers=32, hidden=4096, inter=14336, q=4096, kv=1024, vocab=128256),
}


def linear_shape(model: str, slot: str):
    """(N, K) of one decode linear."""
    c = MODELS[model]
    h, i = c["hidden"], c["inter"]
    return {
        "q": (c["q"], h), "k": (c["kv"], h), "v": (c["kv"], h), "o": (h, c["q"]),
        "gate": (i, h), "up": (i, h), "down": (h, i), "lm_head": (c["vocab"], h),
    }[slot]


def seed_for(config: int, layer: int, slot: str, activation: bool = False) -> int:
    return BASE_SEED + 1000 * config + 16 * layer + SLOT_ID[slot] + (8 if activation else 0)


def _gen(seed: int) -> torch.Generator:
    g = torch.Generator(device="cpu")
    g.manual_seed(int(seed))
    return g


def weight(n: int, k: int, seed: int, std: float = 0.02, row_gain_sigma: float = 0.5) -> torch.Tensor:
    """N(0, std^2) x per-row log-normal gain, rounded to bf16.  [n, k] CPU bf16."""
    g = _gen(seed)
    w = torch.randn(n, k, generator=g, dtype=torch.float32) * std
    gain = torch.exp(torch.randn(n, 1, generator=g, dtype=torch.float32) * row_gain_sigma)
    return (w * gain).to(torch.bfloat16)


def activation(m: int, k: int, seed: int, kind: str = "rmsnorm") -> torch.Tensor:
    """Decode-time activations, [m, k] CPU bf16.

    kind="rmsnorm": N(0,1) x per-channel |N(1, 0.2)| gain, with 0.1% fixed outlier
                    channels x20 (LLM.int8-style outliers).
    kind="swiglu":  silu(a) * b with a, b ~ N(0,1) (the down_proj input).
    """
    g = _gen(seed)
    if kind == "swiglu":
        a = torch.randn(m, k, generator=g, dtype=torch.float32)
        b = torch.randn(m, k, generator=g, dtype=torch.float32)
        return (torch.nn.functional.silu(a) * b).to(torch.bfloat16)
    x = torch.randn(m, k, generator=g, dtype=torch.float32)
    gain = (1.0 + 0.2 * torch.randn(1, k, generator=g, dtype=torch.float32)).abs()
    n_out = max(1, k // 1000)
    idx = torch.randperm(k, generator=g)[:n_out]
    gain[0, idx] *= 20.0
    return (x * gain).to(torch.bfloat16)


def activation_kind(slot: str) -> str:
    return "swiglu" if slot == "down" else "rmsnorm"


def adversarial_weight(n: int, k: int, seed: int) -> torch.Tensor:
    """Blocks that stress the quantiser's conventions (SURVEY §8(c) adversarial list):
    +-equal maxima at various indices, zero / -0 blocks, a single non-zero,
    tiny (fp16-subnormal d) and large blocks, exact half-way quotients."""
    g = _gen(seed)
    w = (torch.randn(n, k, generator=g, dtype=torch.float32) * 0.02)
    G = k // 32
    blocks = w.view(n, G, 32)
    kinds = torch.randint(0, 8, (n, G), generator=g)
    for r in range(n):
        for gi in range(G):
            t = int(kinds[r, gi])
            b = blocks[r, gi]
            if t == 0:      # +a and -a, equal magnitude, first index decides the sign of d
                i, j = torch.randperm(32, generator=g)[:2].tolist()
                a = float(b.abs().max()) * 1.5 + 0.01
                b[i], b[j] = a, -a
            elif t == 1:    # all zero
                b.zero_()
            elif t == 2:    # negative zeros
                b.copy_(torch.full((32,), -0.0))
            elif t == 3:    # single non-zero
                b.zero_()
                b[int(torch.randint(0, 32, (1,), generator=g))] = float(torch.randn(1, generator=g))
            elif t == 4:    # tiny: fp16-subnormal d
                b.mul_(1e-4)
            elif t == 5:    # large, still far from the fp16 overflow of d
                b.mul_(1e4)
            elif t == 6:    # exact half-way quotients: x = (k + 0.5) * d with d = 1/8
                ks = torch.randint(-8, 8, (32,), generator=g).float()
                b.copy_((ks + 0.5) * 0.125)
                b[0] = -1.0         # m = -1 -> d = 0.125 exactly
            # t == 7: plain gaussian
    return w.to(torch.bfloat16)


def adversarial_activation(m: int, k: int, seed: int) -> torch.Tensor:
    """Groups with amax = 0, x = +-amax, exact half-way x/s, outlier channels."""
    g = _gen(seed)
    x = torch.randn(m, k, generator=g, dtype=torch.float32)
    G = k // 32
    xv = x.view(m, G, 32)
    kinds = torch.randint(0, 5, (m, G), generator=g)
    for i in range(m):
        for gi in range(G):
            t = int(kinds[i, gi])
            b = xv[i, gi]
            if t == 0:
                b.zero_()
            elif t == 1:      # amax = 127 -> s = 1, codes = rounded x
                b.copy_(torch.randint(-1270, 1271, (32,), generator=g).float() / 10.0)
                b[0] = 127.0
            elif t == 2:      # +amax and -amax both present
                b[3] = 4.0
                b[17] = -4.0
            elif t == 3:      # x100 outlier channel
                b[int(torch.randint(0, 32, (1,), generator=g))] *= 100.0
    return x.to(torch.bfloat16)


def wide_range_activation(m: int, k: int, seed: int) -> torch.Tensor:
    """Every 32-group spans ~14 binades (|x| from 2^-14 to 1, random signs) plus one x100
    outlier: stresses fp32 cancellation in offset-code W4A16 accumulation."""
    g = _gen(seed)
    mag = torch.exp2(-14.0 * torch.rand(m, k, generator=g))
    sgn = torch.where(torch.rand(m, k, generator=g) < 0.5, -1.0, 1.0)
    x = (mag * sgn).view(m, k // 32, 32)
    idx = torch.randint(0, 32, (m, k // 32, 1), generator=g)
    x.scatter_(2, idx, x.gather(2, idx) * 100.0)
    return x.view(m, k).to(torch.bfloat16)


def bf16_to_f32_numpy(t: torch.Tensor):
    """Exact widening for the oracle (bf16 -> fp32 is exact)."""
    return t.float().numpy()
