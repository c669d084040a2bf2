"""Pins for the oracle's greedy decode (NEXT-2, "decode uses greedy
(argmax) sampling throughout"): argmax_first against numpy's argmax (a library
routine with the same first-index tie rule), hand-written tie / signed-zero cases, and
the sharding invariant (any P: the sharded winner is the global first maximum)."""
import numpy as np
import pytest


def test_matches_numpy_argmax_random(orc):
    rng = np.random.default_rng(7)
    y = rng.standard_normal((5, 3001)).astype(np.float32)
    assert np.array_equal(orc.argmax_first(y), np.argmax(y, axis=1))


def test_ties_take_the_first_index(orc):
    y = np.array([1.0, 3.0, -2.0, 3.0, 3.0], dtype=np.float32)
    assert orc.argmax_first(y) == 1
    assert orc.argmax_first(np.full(9, 0.25, np.float32)) == 0
    assert orc.argmax_first(np.array([-5.0, -1.0, -1.0], np.float32)) == 1


def test_signed_zero_ties(orc):
    # IEEE comparison: -0.0 == +0.0, so the first of them wins
    assert orc.argmax_first(np.array([-1.0, -0.0, 0.0], np.float32)) == 1
    assert orc.argmax_first(np.array([-1.0, 0.0, -0.0], np.float32)) == 1


def test_quantised_logits_with_many_ties(orc):
    rng = np.random.default_rng(8)
    y = np.round(rng.standard_normal((4, 2000)) * 2).astype(np.float32)   # heavy ties
    assert np.array_equal(orc.argmax_first(y), np.argmax(y, axis=1))


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_colshard_argmax_equals_global(orc, world):
    rng = np.random.default_rng(9 + world)
    y = np.round(rng.standard_normal((3, 4096)) * 3).astype(np.float32)
    y[1, 4095] = y[1].max() + 1            # the winner in the last shard
    y[2, :] = 0.0                          # all tied: index 0
    assert np.array_equal(orc.colshard_argmax(y, world), np.argmax(y, axis=1))
