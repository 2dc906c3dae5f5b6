"""Seeded synthetic inputs shared by the oracle tests and the GPU path's tests/bench.

This module holds NO arithmetic of the method (no topology, no update, no mixing).
It only defines the counter-based input hash and the gradient-bank recipe that
DESIGN.md §"Input recipe" states (SURVEY.md §8(d) "Synthetic inputs"):

    H(seed, tag, row, j) = element c of the SplitMix64 stream of `seed`,
        c  = ((tag << 20) + row) * d + j            (mod 2**64)
        z  = mix64(seed + (c + 1) * 0x9E3779B97F4A7C15)   (mod 2**64)
        v  = (z >> 40) * 2**-23 - 1                 in [-1, 1), exact in fp32

The CUDA library implements the same definition independently in
`cs_synth_fill` (test/bench input generator only); the two are compared
bit-for-bit in tests/test_gpu_parity.py::test_synth_generator_bit_exact.  SplitMix64
is pinned to Vigna's reference outputs in tests/test_oracle_rng.py.

Recipe (all configs):
  x_i^0[j] = H(seed, TAG_INIT, i, j)                     (distinct per worker)
  m^0 = 0, w^0 = 1
  bank[r][j] = H(seed, TAG_GRAD, r, j) * 2**-4,  r in [0, B), B = n + 1
  g_i^t = bank[(t + i) mod B]   (a contiguous [n, d] window of concat(bank, bank[:n]))
  lr = 2**-6, momentum = fp32(0.96), seed = 0
"""
from __future__ import annotations

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
MIX1 = np.uint64(0xBF58476D1CE4E5B9)
MIX2 = np.uint64(0x94D049BB133111EB)

TAG_INIT = 0
TAG_GRAD = 1
ROW_BITS = 20          # rows per tag in the counter layout (max 2**20 rows)
GRAD_SCALE = np.float32(2.0 ** -4)

DEFAULT_LR = np.float32(2.0 ** -6)
DEFAULT_MOMENTUM = np.float32(0.96)


def splitmix64_mix(z: np.ndarray) -> np.ndarray:
    """mix64 finaliser of SplitMix64 (Steele, Lea, Flood 2014; Vigna's splitmix64.c)."""
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * MIX1
        z = (z ^ (z >> np.uint64(27))) * MIX2
    return z ^ (z >> np.uint64(31))


def splitmix64_stream(seed: int, counters: np.ndarray) -> np.ndarray:
    """Element c (0-based) of the SplitMix64 output stream started at `seed`."""
    c = np.asarray(counters, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed & 0xFFFFFFFFFFFFFFFF) + (c + np.uint64(1)) * GOLDEN
    return splitmix64_mix(z)


def hash_uniform(seed: int, tag: int, row: int, d: int, cols: np.ndarray | None = None) -> np.ndarray:
    """H(seed, tag, row, j) for j in `cols` (default: all of [0, d)), as fp32 in [-1, 1)."""
    if cols is None:
        cols = np.arange(d, dtype=np.uint64)
    cols = np.asarray(cols, dtype=np.uint64)
    with np.errstate(over="ignore"):
        base = (np.uint64(tag) << np.uint64(ROW_BITS)) + np.uint64(row)
        c = base * np.uint64(d) + cols
    z = splitmix64_stream(seed, c)
    v = (z >> np.uint64(40)).astype(np.float64) * (2.0 ** -23) - 1.0
    return v.astype(np.float32)  # exact: 24-bit integer times a power of two


def init_params(seed: int, rows, d: int, cols=None) -> np.ndarray:
    """x^0 rows (global worker ids `rows`) restricted to `cols`."""
    return np.stack([hash_uniform(seed, TAG_INIT, int(r), d, cols) for r in rows])


def grad_bank(seed: int, n: int, d: int, cols=None) -> np.ndarray:
    """bank[r] for r in [0, n+1): fp32 [B, len(cols)], scaled by 2**-4 (exact)."""
    B = n + 1
    return np.stack([hash_uniform(seed, TAG_GRAD, r, d, cols) * GRAD_SCALE for r in range(B)])


def grads_at(bank: np.ndarray, n: int, t: int, rows=None) -> np.ndarray:
    """g^t for workers `rows` (default all n): row i takes bank[(t + i) mod B]."""
    B = bank.shape[0]
    rows = range(n) if rows is None else rows
    return bank[[(t + i) % B for i in rows]]


def sample_columns(d: int, bounds, stride: int = 1024, seed: int = 0) -> np.ndarray:
    """Columns for sampled full-size parity: every segment boundary (±2), a stride, the tail."""
    cols = set(range(0, d, stride))
    for b in bounds:
        for off in (-2, -1, 0, 1, 2):
            j = int(b) + off
            if 0 <= j < d:
                cols.add(j)
    cols.update(range(max(0, d - 8), d))
    rng = np.random.default_rng(seed)
    cols.update(int(c) for c in rng.integers(0, d, size=min(d, 256)))
    return np.array(sorted(cols), dtype=np.int64)


def resnet50_layers():
    """ResNet-50's parameter tensors in definition order (the
    paper's model and its "blocks and FC layer" segments).  Shapes follow the
    architecture (He et al. 2016; torchvision layout): stem conv 7x7/64 + BN, four
    stages of [3, 4, 6, 3] bottlenecks (1x1, 3x3, 1x1 convs, expansion 4, a 1x1
    projection + BN in each stage's first block), FC 2048 -> 1000.  BN running
    statistics are buffers, not parameters.

    Returns (sizes, block): element count of each of the 161 tensors and its block
    id (0 = stem, 1..16 = bottleneck blocks, 17 = FC).  Structure only, no values."""
    sizes, block = [], []

    def conv_bn(cin, cout, kk, b):
        sizes.extend([cout * cin * kk * kk, cout, cout])  # conv weight, BN weight, BN bias
        block.extend([b, b, b])

    conv_bn(3, 64, 7, 0)
    cin, b = 64, 0
    for stage, (blocks, width) in enumerate(zip([3, 4, 6, 3], [64, 128, 256, 512])):
        for i in range(blocks):
            b += 1
            conv_bn(cin, width, 1, b)
            conv_bn(width, width, 3, b)
            conv_bn(width, width * 4, 1, b)
            if i == 0:
                conv_bn(cin, width * 4, 1, b)  # projection shortcut
            cin = width * 4
    sizes.extend([1000 * 2048, 1000])
    block.extend([b + 1, b + 1])
    return sizes, block
