"""bf16 wire format for exchanged segments (the
paper trained in mixed precision).  Test infrastructure only.

Reading C-20: the master state stays fp32; what a worker RECEIVES (the
sender's post-update segment y, Alg. 1 l.8) is the sender's value rounded to the
nearest bf16 (8-bit significand, ties to even) and widened back to fp32 exactly.  The
worker's own y and the push-sum weights are not rounded:

    x'_i = fl(fl(y_i + bf16(y_src(i))) * 0.5),   w'_i unchanged from the fp32 rule.

It applies to every received segment, on the same GPU or not, so the result does not
depend on how workers are placed on GPUs.
"""
from __future__ import annotations

import numpy as np


def bf16_round(v: np.ndarray) -> np.ndarray:
    """Round fp32 values to the nearest bf16 (ties to even), returned as fp32.

    Written out on the bit pattern: keep the top 16 bits, adding half an ulp of the kept
    part (0x7FFF) plus the kept part's lowest bit so exact halves go to the even one.
    Finite inputs only (the step flags non-finite gradients)."""
    u = np.ascontiguousarray(v, dtype=np.float32).view(np.uint32).astype(np.uint64)
    r = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return r.astype(np.uint32).view(np.float32)
