"""Optimizer steps for the block parameters — plain fp64 definitions.  TEST
INFRASTRUCTURE ONLY (same import rule as the rest of oracle/).

The paper updates the expert parameters as soon as their gradients are final (at
E_1^l of the backward) and the replicated MHA/gate parameters after their
all-reduce; it does not name the optimizer (reading Q17), so the library
offers the two usual ones, written out here exactly as stated:

* SGD with momentum and L2 weight decay (the PyTorch `torch.optim.SGD` form):
      d = g + wd·w;   b = μ·b + d   (b = d at step 1);   w = w − lr·b
* AdamW (Loshchilov & Hutter, decoupled weight decay; the PyTorch `AdamW` form):
      m = β1·m + (1−β1)·g;   v = β2·v + (1−β2)·g²
      m̂ = m / (1−β1^t);   v̂ = v / (1−β2^t)
      w = w·(1 − lr·wd) − lr·m̂ / (√v̂ + ε)
"""
from __future__ import annotations

import numpy as np


def sgd_momentum_step(w, b, g, *, lr, momentum, weight_decay, step):
    """One SGD step; returns (w, b) as new fp64 arrays."""
    w, b, g = (np.asarray(a, dtype=np.float64) for a in (w, b, g))
    d = g + weight_decay * w
    b = d.copy() if step == 1 else momentum * b + d
    return w - lr * b, b


def adamw_step(w, m, v, g, *, lr, beta1, beta2, eps, weight_decay, step):
    """One AdamW step; returns (w, m, v) as new fp64 arrays."""
    w, m, v, g = (np.asarray(a, dtype=np.float64) for a in (w, m, v, g))
    m = beta1 * m + (1.0 - beta1) * g
    v = beta2 * v + (1.0 - beta2) * g * g
    mh = m / (1.0 - beta1 ** step)
    vh = v / (1.0 - beta2 ** step)
    w = w * (1.0 - lr * weight_decay) - lr * mh / (np.sqrt(vh) + eps)
    return w, m, v
