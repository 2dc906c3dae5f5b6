"""Communication-interval mode: accumulate the gradient over I local micro-steps,
then one gossip round with the mean.  Test infrastructure only.

PAPER.md:209 (section 4): "we chose to increase the communication interval and
accumulate the loss during this interval instead of increasing the physical
scale"; Table 1: "Communication Interval 42".  The state machine is
SPEC.md:395-398 accumulate_and_flush:

    accumulator += grad; count += 1;
    when count reaches comm_interval: emit accumulator / comm_interval and reset;
    otherwise emit nothing.

Accumulating the loss over I micro-batches and back-propagating once gives the
same gradient as accumulating the I per-micro-batch gradients (linearity of the
derivative), so the accumulator holds gradients.  Arithmetic is in the dtype of
the inputs, one rounding per operation (fp32 for kernel parity, fp64 for the
closed-form pins); the accumulator starts at +0.0 and the mean is a true division
(reading C-17).
"""
from __future__ import annotations

import numpy as np


class Accumulator:
    """SPEC WorkerState's (accumulator, count) pair for one or more workers."""

    def __init__(self, shape, interval: int, dtype=np.float32):
        if interval < 1:
            raise ValueError("comm_interval must be >= 1")
        self.interval = int(interval)
        self.dtype = np.dtype(dtype)
        self.acc = np.zeros(shape, dtype=self.dtype)
        self.count = 0

    def push(self, grad):
        """accumulate_and_flush(state, grad) -> the mean gradient, or None."""
        grad = np.asarray(grad)
        assert grad.dtype == self.dtype and grad.shape == self.acc.shape
        self.acc = self.acc + grad
        self.count += 1
        if self.count == self.interval:
            out = self.acc / self.dtype.type(self.interval)
            self.acc = np.zeros_like(self.acc)
            self.count = 0
            return out
        return None
