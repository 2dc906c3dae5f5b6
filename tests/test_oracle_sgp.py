"""Pins for oracle/sgp.py: SPEC's worked examples, the inverse
relation, and the exact averaging the exponential graph reaches in log2 n rounds."""
import numpy as np
import pytest

from oracle.gossip import gossip_step
from oracle.sgp import exponential_peer, exponential_topology

F32 = np.float32


def test_spec_examples():
    assert exponential_peer(0, 0, 8) == 1
    assert exponential_peer(0, 2, 8) == 4
    assert exponential_peer(5, 3, 8) == 6
    with pytest.raises(ValueError):
        exponential_peer(0, 0, 6)
    with pytest.raises(ValueError):
        exponential_topology(0, 1, 1)


@pytest.mark.parametrize("n", [2, 4, 8, 64, 1024])
def test_topology_is_the_inverse_of_the_peer_map_and_a_derangement(n):
    for t in range(12):
        src = exponential_topology(t, n, 3)
        assert np.all(src == src[0])
        for i in range(n):
            assert exponential_peer(int(src[0, i]), t, n) == i
        assert sorted(src[0].tolist()) == list(range(n)) and np.all(src[0] != np.arange(n))


@pytest.mark.parametrize("n", [2, 4, 8, 16])
def test_exact_average_after_log2_n_rounds(n):
    # x_i <- (x_i + x_{i - 2^j}) / 2 for j = 0..log2 n - 1 gives every worker the mean of all
    # n rows (sum over all offsets 0..n-1); dyadic inputs keep every step exact in fp32
    rng = np.random.default_rng(n)
    d = 40
    x = (rng.integers(-512, 512, size=(n, d)) * 2.0 ** -6).astype(F32)
    mean = x.astype(np.float64).mean(axis=0)
    w = np.ones((n, 1), F32)
    seg = np.zeros(d, dtype=np.int64)
    z = np.zeros_like(x)
    for t in range(n.bit_length() - 1):
        x, _, w = gossip_step(x, z, z, w, exponential_topology(t, n, 1), seg, 0.0, 0.0)
    assert np.array_equal(x, np.broadcast_to(mean.astype(F32), x.shape))
    assert np.all(w == 1)


@pytest.mark.parametrize("n", [2, 8, 32])
def test_peer_offsets_cycle_through_powers_of_two(n):
    # the send offset at round t is 2^(t mod log2 n), so rounds 0..log2 n - 1
    # use the distinct offsets 1, 2, 4, ..., n/2 and the schedule repeats with period log2 n
    L = n.bit_length() - 1
    offs = [(exponential_peer(0, t, n) - 0) % n for t in range(3 * L)]
    assert offs[:L] == [1 << j for j in range(L)]
    assert offs == offs[:L] * 3
    for t in range(L):
        assert np.array_equal(exponential_topology(t, n, 2), exponential_topology(t + L, n, 2))
