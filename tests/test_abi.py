"""CPU tests of the C-ABI boundary: the library builds for sm_100a, loads, exports
every symbol include/mcapq.h declares, and its host logic (validation, status
codes, profile JSON -> routes) behaves as documented.  No kernel is launched."""
import ctypes
import json
import math
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "mcapq.h")
GOLD = os.path.join(ROOT, "tests", "golden")


@pytest.fixture(scope="module")
def L():
    from paper_2604_21026_b200 import build, _lib
    build.build()
    return _lib.load()


def _declared():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(mcapq_[a-z0-9_]+)\s*\(", text)))


def test_every_declared_symbol_is_exported(L):
    from paper_2604_21026_b200 import _lib
    names = _declared()
    assert len(names) >= 30
    for n in names:
        assert hasattr(L, n), n
    assert sorted(_lib.SIGNATURES) == names      # the binding mirrors the header one for one


def test_sass_is_sm100a_and_uses_int8_bf16_tensor_and_dp4a(L):
    from paper_2604_21026_b200 import _lib
    out = subprocess.run(["cuobjdump", "-sass", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    assert "sm_100a" in out or "SM100" in out.upper()
    for mnem in ("IDP.4A", "IMMA.16832", "HMMA.16816.F32.BF16", "PREEXIT", "ACQBULK"):
        assert mnem in out, mnem
    # no generic compute_100 PTX (which would reject the sm_100a-only features)
    ptx = subprocess.run(["cuobjdump", "-lptx", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    assert "compute_100 " not in ptx


def test_status_strings(L):
    assert L.mcapq_abi_version() == 1
    assert L.mcapq_status_string(0) == b"ok"
    assert L.mcapq_status_string(8) == b"workspace too small"


def test_sizes(L):
    assert L.mcapq_w4_nib_bytes(4096, 14336) == 4096 * 7168
    assert L.mcapq_w4_scale_bytes(4096, 14336) == 4096 * 448 * 2
    # 18 bytes per 32 weights
    assert (L.mcapq_w4_nib_bytes(7, 64) + L.mcapq_w4_scale_bytes(7, 64)) == 7 * 2 * 18
    assert L.mcapq_workspace_bytes(1, 1, 10, 64) == 0            # W4A16 needs none
    assert L.mcapq_workspace_bytes(0, 2, 10, 64) >= 2 * 64 + 2 * 2 * 8


def test_validation_happens_before_any_launch(L):
    P = ctypes.c_void_p
    fake = P(0x1000)          # 16-byte aligned, never dereferenced: validation fails first
    # K % 32 != 0
    st = L.mcapq_w4a16(fake, fake, 8, 48, fake, 1, 48, fake, 0, 8, None)
    assert st == 1 and b"k%32" in L.mcapq_last_error() or b"shape" in L.mcapq_last_error()
    # NULL pointer
    assert L.mcapq_w4a16(None, fake, 8, 64, fake, 1, 64, fake, 0, 8, None) == 1
    # misaligned
    assert L.mcapq_w4a16(P(0x1001), fake, 8, 64, fake, 1, 64, fake, 0, 8, None) == 1
    # bad dtype
    assert L.mcapq_w4a16(fake, fake, 8, 64, fake, 1, 64, fake, 7, 8, None) == 2
    # ldy too small
    assert L.mcapq_w4a16(fake, fake, 16, 64, fake, 1, 64, fake, 0, 8, None) == 1
    # workspace too small
    assert L.mcapq_w4a8_x(fake, fake, 8, 64, fake, 1, 64, fake, 0, 8, fake, 16, None) == 8
    # bad route
    assert L.mcapq_linear(5, fake, fake, 8, 64, fake, 1, 64, fake, 0, 8, fake, 4096, None) == 1
    # M < 1
    assert L.mcapq_w4a8(fake, fake, 8, 64, fake, fake, fake, 0, fake, 0, 8, None) == 1


def _routes(L, text, tau=float("nan")):
    from paper_2604_21026_b200 import _lib
    h = ctypes.c_void_p()
    b = text.encode()
    st = L.mcapq_profile_parse(b, len(b), tau, ctypes.byref(h))
    if st != 0:
        return st, None, None
    n = L.mcapq_profile_layers(h)
    r = (ctypes.c_uint8 * n)()
    s = (ctypes.c_double * n)()
    assert L.mcapq_profile_routes(h, ctypes.cast(r, ctypes.c_void_p), n) == 0
    assert L.mcapq_profile_scores(h, ctypes.cast(s, ctypes.c_void_p), n) == 0
    assert L.mcapq_profile_routes(h, ctypes.cast(r, ctypes.c_void_p), n + 1) == 1
    tau_out = L.mcapq_profile_tau(h)
    L.mcapq_profile_free(h)
    return 0, list(r), (list(s), tau_out)


def test_profile_golden_matches_oracle(L, orc):
    # a7 parity: the library's dispatch table equals the oracle's on the paper's vector
    text = open(os.path.join(GOLD, "llama32_1b_profile.json")).read()
    st, routes, (scores, tau) = _routes(L, text)
    assert st == 0 and tau == 0.7
    o_scores, o_tau, o_routes = orc.routes_from_profile(text)
    assert routes == o_routes == [0] * 15 + [1]
    assert scores == o_scores
    for t in (2.0, 0.30, 0.10, 0.05, 0.0, 0.7, 0.699, 0.475):
        assert _routes(L, text, t)[1] == orc.route_layers(o_scores, t)


def test_profile_raw_scores_and_degenerate(L, orc):
    obj = json.load(open(os.path.join(GOLD, "llama32_1b_profile.json")))
    del obj["scores"]
    text = json.dumps(obj)
    st, routes, (scores, _) = _routes(L, text)
    o_scores, _, o_routes = orc.routes_from_profile(text)
    assert routes == o_routes
    assert all(abs(a - b) <= 1e-15 for a, b in zip(scores, o_scores))
    st, routes, _ = _routes(L, json.dumps({"raw_scores": [7.0] * 28}))
    assert routes == [0] * 28


@pytest.mark.parametrize("bad,code", [
    ("[1,2]", 4), ("{\"tau\": 0.5}", 4), ("{\"scores\": [0.1, 1.5]}", 4),
    ("{\"scores\": [0.1, 0.2], \"num_layers\": 3}", 4), ("{\"scores\": [0.1,", 4),
    ("{\"scores\": [0.1, 0.2]} x", 4), ("{\"scores\": [0.5], \"tau\": -1}", 3),
    ("{\"scores\": [\"a\"]}", 4),
    ("{\"raw_scores\": [1.0, 2.0], \"epsilon\": 0}", 4), ("{\"raw_scores\": [1.0, 2.0], \"epsilon\": -1e-9}", 4),
    ("{\"raw_scores\": [1.0, -2.0]}", 4),
])
def test_profile_errors(L, bad, code):
    assert _routes(L, bad)[0] == code


def test_profile_ignores_unknown_keys(L):
    text = json.dumps({"arch": "x", "nested": {"a": [1, {"b": None}], "t": True}, "scores": [0.2, 0.9], "tau": 0.5})
    assert _routes(L, text)[1] == [0, 1]


def _write(L, raw, prompts, tau):
    buf = ctypes.create_string_buffer(1 << 16)
    n = ctypes.c_size_t()
    arr = (ctypes.c_double * len(raw))(*raw)
    st = L.mcapq_profile_write_json(ctypes.cast(arr, ctypes.c_void_p), len(raw), prompts, tau, buf, len(buf),
                                    ctypes.byref(n))
    return st, buf.value.decode()


def test_profile_writer_canonical_round_trip(L):
    """The artifact mcapq_profile_write_json emits is canonical: keys sorted, every double in
    its shortest round-trip form -- so parse(text) reproduces the raw scores exactly and
    writing them again gives the same bytes (serialise -> load -> serialise identity)."""
    raw = [85.14, 117.62, 61.0, 0.1 + 0.2, 1e-300, 142.0, 3.0000000000000004, 0.0]
    st, text = _write(L, raw, 12, 0.7)
    assert st == 0
    obj = json.loads(text)
    assert list(obj) == sorted(obj)
    assert obj["raw_scores"] == raw and obj["tau"] == 0.7
    assert text == json.dumps(obj, separators=(",", ":"))           # Python's repr is also shortest round-trip
    st2, text2 = _write(L, obj["raw_scores"], obj["prompt_count"], obj["tau"])
    assert st2 == 0 and text2 == text
    assert _routes(L, text)[0] == 0
    assert _write(L, [1.0, -1.0], 1, 0.7)[0] == 1                    # negative raw scores are rejected
