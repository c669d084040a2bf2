"""NEXT-3: MCAP profiling (Alg. 1, sec:mcap P:533-559) -- oracle pins (CPU), the
profile-artifact writer round trip (host logic, CPU) and the GPU accumulator vs the oracle."""
import json
import os

import numpy as np
import pytest
import torch

import oracle

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "llama32_1b_profile.json")


# ---------------------------------------------------------------- oracle pins (closed forms)
def test_mcap_oracle_pythagorean_tokens():
    # q = (3, 0..), v = (4, 0..) -> ||[q, v]|| = 5;  ffn = (12, 5, 0..) -> 13;  token t scaled by t + 1
    m = 4
    q = np.zeros((m, 8)); v = np.zeros((m, 3)); f = np.zeros((m, 6))
    for t in range(m):
        q[t, 0], v[t, 2], f[t, 1], f[t, 4] = 3 * (t + 1), 4 * (t + 1), 12 * (t + 1), 5 * (t + 1)
    (s,) = oracle.mcap_raw_scores([[(q, v, f)]])
    assert s == pytest.approx(18.0 * (m + 1) / 2, rel=0, abs=1e-12)


def test_mcap_oracle_mean_of_prompt_means():
    # line 10 averages per-prompt token means (1/k sum_j 1/|p_j| sum_t), not all tokens pooled
    one = lambda m, a: (np.full((m, 1), a), np.zeros((m, 1)), np.zeros((m, 1)))   # noqa: E731
    (s,) = oracle.mcap_raw_scores([[one(1, 1.0)], [one(3, 3.0)]])
    assert s == pytest.approx(2.0, abs=1e-15)          # (1 + 3) / 2, not (1 + 9) / 4


def test_mcap_oracle_token_permutation_and_layer_independence():
    rng = np.random.default_rng(1)
    lay = [(rng.normal(size=(7, 16)), rng.normal(size=(7, 4)), rng.normal(size=(7, 16))) for _ in range(3)]
    perm = rng.permutation(7)
    s1 = oracle.mcap_raw_scores([lay])
    s2 = oracle.mcap_raw_scores([[(q[perm], v[perm], f[perm]) for q, v, f in lay]])
    assert np.allclose(s1, s2, rtol=1e-14, atol=0)
    s3 = oracle.mcap_raw_scores([[lay[1]]])
    assert s3[0] == pytest.approx(s1[1], rel=1e-15)


def test_mcap_outlier_layer_routes_to_w4a16():
    # the paper's reading of the score: the layer with the largest activation
    # range is the one that cannot absorb INT8 error -> the only W4A16 layer at tau = 0.7
    rng = np.random.default_rng(2)
    layers = []
    for i in range(5):
        g = 20.0 if i == 3 else 1.0
        layers.append((rng.normal(size=(9, 32)) * g, rng.normal(size=(9, 8)), rng.normal(size=(9, 32)) * g))
    s = oracle.mcap_raw_scores([layers])
    assert oracle.route_layers(oracle.minmax_normalize(s)) == [0, 0, 0, 1, 0]


# ---------------------------------------------------------------- artifact writer (host logic)
def test_profile_write_json_round_trip_golden():
    mq = pytest.importorskip("paper_2604_21026_b200")
    mq.load()
    g = json.load(open(GOLD))
    text = mq.profile_write_json(g["raw_scores"], g["prompt_count"], g["tau"])
    obj = json.loads(text)
    assert obj["raw_scores"] == g["raw_scores"] and obj["num_layers"] == 16 and obj["prompt_count"] == 12
    p = mq.profile_parse(text)
    _, _, routes = oracle.routes_from_profile(text)
    assert list(p.routes()) == list(routes) == [0] * 15 + [1]      # tab:per_layer_scores -> {15}
    assert np.array_equal(np.array(p.scores()), np.array(oracle.minmax_normalize(g["raw_scores"])))


def test_profile_write_json_errors():
    mq = pytest.importorskip("paper_2604_21026_b200")
    mq.load()
    with pytest.raises(mq.McapqError):
        mq.profile_write_json([1.0, float("nan")], 1)
    with pytest.raises(mq.McapqError):
        mq.profile_write_json([], 1)


# ---------------------------------------------------------------- GPU accumulator vs the oracle
def _synthetic_prompts(L, lens, seed):
    """Seeded bf16 linear outputs of L layers for prompts of the given lengths; layer L-2
    carries 0.1 % outlier channels x20 (LLM.int8-style)."""
    g = torch.Generator().manual_seed(seed)
    prompts = []
    for m in lens:
        layers = []
        for i in range(L):
            scale = 1.0 + 0.1 * i
            q = torch.randn(m, 2048, generator=g) * scale
            v = torch.randn(m, 512, generator=g) * scale
            f = torch.randn(m, 2048, generator=g) * scale * 0.5
            if i == L - 2:
                q[:, :8] *= 20
                f[:, :8] *= 20
            layers.append((q.bfloat16(), v.bfloat16(), f.bfloat16()))
        prompts.append(layers)
    return prompts


@pytest.mark.gpu
def test_mcap_accumulate_vs_oracle_and_routes():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2604_21026_b200 as mq
    mq.load()
    L, lens = 6, (5, 17, 40)
    prompts = _synthetic_prompts(L, lens, 2604)
    k = len(prompts)
    score = torch.zeros(L, dtype=torch.float64, device="cuda")
    for layers in prompts:
        for i, (q, v, f) in enumerate(layers):
            m = q.shape[0]
            mq.mcap_accumulate(q.cuda(), v.cuda(), f.cuda(), 1.0 / (k * m), score[i:i + 1])
    got = score.cpu().numpy()
    ref = np.array(oracle.mcap_raw_scores([[(q.float().numpy(), v.float().numpy(), f.float().numpy())
                                             for q, v, f in layers] for layers in prompts]))
    assert np.allclose(got, ref, rtol=1e-12, atol=0), (got, ref)
    text = mq.profile_write_json(list(got), k, 0.7)
    routes = list(mq.profile_parse(text).routes())
    assert routes == oracle.route_layers(oracle.minmax_normalize(list(ref)))
    assert routes[L - 2] == 1 and sum(routes) == 1
    # deterministic: a second pass gives the same bits
    again = torch.zeros(L, dtype=torch.float64, device="cuda")
    for layers in prompts:
        for i, (q, v, f) in enumerate(layers):
            mq.mcap_accumulate(q.cuda(), v.cuda(), f.cuda(), 1.0 / (k * q.shape[0]), again[i:i + 1])
    assert torch.equal(again, score)


@pytest.mark.gpu
def test_mcap_accumulate_strided_rows():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2604_21026_b200 as mq
    mq.load()
    g = torch.Generator().manual_seed(7)
    big = torch.randn(9, 3000, generator=g).bfloat16()
    q, v, f = big[:, :2048], big[:, 2048:2560], big[:, 512:2560]       # views with ld = 3000
    score = torch.zeros(1, dtype=torch.float64, device="cuda")
    bd = big.cuda()
    mq.mcap_accumulate(bd[:, :2048], bd[:, 2048:2560], bd[:, 512:2560], 0.5, score)
    (ref,) = oracle.mcap_raw_scores([[(q.float().numpy(), v.float().numpy(), f.float().numpy())]])
    assert score.item() == pytest.approx(0.5 * 9 * ref, rel=1e-12)
