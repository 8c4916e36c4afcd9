"""Model edges around the block stack — plain fp64 definitions.  TEST INFRASTRUCTURE
ONLY (same import rule as the rest of oracle/).

* Token embedding (the model input of the paper's GPT2/BERT/LLaMA-shaped models,
  SURVEY §8(f) #4): x[t] = table[ids[t]]; its gradient scatters dx back,
  dtable[v] = Σ_{t: ids[t] = v} dx[t].
* Loss, Eqs.(19)-(23): loss = (1/B) Σ_i ℓ(x_i, y_i), and with R micro-batches
  the scaled per-chunk loss of Eq.(21) is (1/B) Σ_{i in chunk r} ℓ(x_{r,i}, y_{r,i}), so the
  chunk losses add up to the full loss (Eq.(22)) and so do their gradients (Eq.(23)).
  Reading Q18: ℓ is the softmax cross-entropy of one token,
      ℓ_t = log Σ_v exp(l_tv) − l_{t, y_t},   ∂ℓ_t/∂l_tv = softmax(l_t)_v − [v = y_t],
  B counts the labelled tokens, and a token with label < 0 (or ≥ V) carries no loss.
"""
from __future__ import annotations

import numpy as np


def embed_forward(table: np.ndarray, ids: np.ndarray) -> np.ndarray:
    """x[t] = table[ids[t]]; an id outside [0, V) gives a zero row (the library's contract)."""
    V, M = table.shape
    x = np.zeros((len(ids), M))
    for t, v in enumerate(ids):
        if 0 <= v < V:
            x[t] = table[v]
    return x


def embed_backward(ids: np.ndarray, dx: np.ndarray, V: int) -> np.ndarray:
    """dtable[v] = Σ_{t: ids[t] = v} dx[t], summed in t order."""
    d = np.zeros((V, dx.shape[1]))
    for t, v in enumerate(ids):
        if 0 <= v < V:
            d[v] += dx[t]
    return d


def xent(logits: np.ndarray, labels: np.ndarray, scale: float):
    """Per-token losses ℓ_t (0 for unlabelled rows), loss = scale·Σ_t ℓ_t and
    dlogits = scale·(softmax − onehot) (zero rows where unlabelled)."""
    T, V = logits.shape
    losses = np.zeros(T)
    dl = np.zeros((T, V))
    for t in range(T):
        y = int(labels[t])
        if not 0 <= y < V:
            continue
        row = logits[t]
        m = row.max()
        lse = m + np.log(np.exp(row - m).sum())
        losses[t] = lse - row[y]
        p = np.exp(row - lse)
        p[y] -= 1.0
        dl[t] = scale * p
    return losses, scale * losses.sum(), dl


def lm_head_forward(h: np.ndarray, w: np.ndarray) -> np.ndarray:
    """logits[t][v] = Σ_m h[t][m]·W[v][m] (the projection feeding the loss)."""
    return h @ w.T


def lm_head_backward(h: np.ndarray, w: np.ndarray, dlogits: np.ndarray):
    """dh = dlogits·W, dW = dlogitsᵀ·h (the two adjoints of the projection)."""
    return dlogits @ w, dlogits.T @ h
