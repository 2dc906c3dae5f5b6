"""Pins the two counter-based generators against their published known answers."""
import os

import numpy as np

import synth
from conftest import GOLDEN
from oracle.philox import philox4x32_10, philox4x32_10_np


def _kat_lines(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return [ln.split() for ln in f if ln.strip() and not ln.startswith("#")]


def test_philox_random123_kat():
    for row in _kat_lines("philox4x32_10_kat.txt"):
        v = [int(h, 16) for h in row]
        assert philox4x32_10(v[0:4], v[4:6]) == tuple(v[6:10])


def test_philox_vectorised_equals_scalar():
    rng = np.random.default_rng(1)
    c = rng.integers(0, 2**32, size=(4, 64), dtype=np.uint64)
    key = (0x12345678, 0x9ABCDEF0)
    vec = philox4x32_10_np(*c, *key)
    for j in range(64):
        assert philox4x32_10([c[i][j] for i in range(4)], key) == tuple(int(vec[i][j]) for i in range(4))


def test_splitmix64_reference_outputs():
    want = [int(r[0], 16) for r in _kat_lines("splitmix64_kat.txt")]
    got = synth.splitmix64_stream(0, np.arange(len(want)))
    assert [int(v) for v in got] == want


def test_hash_uniform_range_and_exactness():
    v = synth.hash_uniform(0, synth.TAG_INIT, 3, 100_000)
    assert v.dtype == np.float32
    assert v.min() >= -1.0 and v.max() < 1.0
    # every value is k * 2^-23 - 1 for an integer k < 2^24
    k = (v.astype(np.float64) + 1.0) * 2.0**23
    assert np.all(k == np.round(k))
    assert abs(float(v.mean())) < 0.01


def test_hash_uniform_random_access():
    d = 1000
    full = synth.hash_uniform(5, synth.TAG_GRAD, 7, d)
    cols = np.array([0, 17, 999])
    assert np.array_equal(full[cols], synth.hash_uniform(5, synth.TAG_GRAD, 7, d, cols))
