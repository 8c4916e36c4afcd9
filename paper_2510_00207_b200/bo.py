"""Bayesian-optimisation auto-tuner for the all-reduce chunk size S_p (host side).

FlowMoE §4.1 and Appendix D: BO fits a Gaussian process
(Matérn kernel) to measured (S_p, per-iteration time) pairs — each the mean of ~10
iterations — and picks the next S_p by maximising Expected Improvement with ξ = 0.1
(P:1008), starting from one random sample, 8 samples in total, over the
search space (0, max AR tensor bytes per block].  A re-tune is triggered
when |T − F̂(S_p*)| / F̂(S_p*) > δ (Eq.(18); δ not given, default 0.1).
Grid search (8 equal parts) and random search are the paper's baselines.

Fixed GP hyperparameters (8 samples cannot support marginal-likelihood fits):
length scale 0.2 × interval width, signal variance = sample variance of the
observations, noise 1e-6 × signal variance, prior mean = sample mean; EI is
maximised over a 512-point grid of the interval.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Callable

import numpy as np


def matern52(a: np.ndarray, b: np.ndarray, length: float, var: float) -> np.ndarray:
    r = np.abs(a[:, None] - b[None, :]) / length
    s5 = math.sqrt(5.0)
    return var * (1.0 + s5 * r + 5.0 / 3.0 * r * r) * np.exp(-s5 * r)


@dataclass
class GP:
    length: float
    signal_var: float
    noise_var: float
    mean0: float = 0.0
    xs: np.ndarray = field(default_factory=lambda: np.zeros(0))
    ys: np.ndarray = field(default_factory=lambda: np.zeros(0))

    def fit(self, xs, ys):
        self.xs = np.asarray(xs, dtype=np.float64)
        self.ys = np.asarray(ys, dtype=np.float64)
        K = matern52(self.xs, self.xs, self.length, self.signal_var)
        K[np.diag_indices_from(K)] += self.noise_var
        jitter = 0.0
        for _ in range(8):
            try:
                self._L = np.linalg.cholesky(K + jitter * np.eye(len(K)))
                break
            except np.linalg.LinAlgError:
                jitter = max(1e-12, jitter * 10 if jitter else 1e-10 * max(1.0, self.signal_var))
        else:
            raise np.linalg.LinAlgError("GP kernel matrix is singular")
        self._alpha = np.linalg.solve(self._L.T, np.linalg.solve(self._L, self.ys - self.mean0))
        return self

    def posterior(self, q):
        q = np.asarray(q, dtype=np.float64)
        Ks = matern52(q, self.xs, self.length, self.signal_var)
        mu = self.mean0 + Ks @ self._alpha
        v = np.linalg.solve(self._L, Ks.T)
        var = np.maximum(self.signal_var - np.sum(v * v, axis=0), 0.0)
        return mu, var


def expected_improvement(mean, var, best, xi=0.1):
    """EI for minimisation: with σ = √var, z = (best − mean − ξ)/σ,
    EI = (best − mean − ξ)·Φ(z) + σ·φ(z); EI = max(0, best − mean − ξ) when σ = 0."""
    mean = np.asarray(mean, dtype=np.float64)
    sd = np.sqrt(np.maximum(np.asarray(var, dtype=np.float64), 0.0))
    imp = best - mean - xi
    out = np.maximum(imp, 0.0)
    pos = sd > 0
    if np.any(pos):
        z = imp[pos] / sd[pos]
        cdf = 0.5 * (1.0 + np.vectorize(math.erf)(z / math.sqrt(2.0)))
        pdf = np.exp(-0.5 * z * z) / math.sqrt(2.0 * math.pi)
        out = out.astype(np.float64)
        out[pos] = imp[pos] * cdf + sd[pos] * pdf
    return out


@dataclass
class TuneResult:
    best_sp: float
    best_time: float
    log: list  # (round, S_p, observed, incumbent)


def bo_tune(objective: Callable[[float], float], lo: float, hi: float, budget: int = 8,
            xi: float = 0.1, seed: int = 0, candidates: int = 512,
            quantum: float = 1.0, xi_relative: bool = False) -> TuneResult:
    """1 random initial sample, then budget−1 EI-maximising samples on (lo, hi].

    xi is EI's exploration margin in the objective's units (ξ = 0.1, SPEC bo_tuner /
    Appendix D).  xi_relative=True instead scales it by the observed spread (ξ·σ_obs) — a
    design choice for objectives whose units make an absolute 0.1 meaningless (DESIGN.md,
    S_p auto-tuning); tools/tune_sp.py uses it for iteration times in ms."""
    rng = np.random.default_rng(seed)
    grid = lo + (hi - lo) * (np.arange(1, candidates + 1) / candidates)
    xs, ys, log = [], [], []

    def snap(v):
        return float(min(hi, max(quantum, math.ceil(v / quantum) * quantum)))

    x0 = snap(lo + (hi - lo) * rng.uniform(1e-9, 1.0))
    for rnd in range(budget):
        x = x0 if rnd == 0 else None
        if x is None:
            ya = np.asarray(ys)
            sv = float(np.var(ya)) if len(ya) > 1 and np.var(ya) > 0 else max(1e-12, float(np.mean(np.abs(ya))) * 1e-2)
            gp = GP(length=0.2 * (hi - lo), signal_var=sv, noise_var=1e-6 * sv, mean0=float(np.mean(ya))).fit(xs, ya)
            mu, var = gp.posterior(grid)
            ei = expected_improvement(mu, var, float(np.min(ya)), xi * math.sqrt(sv) if xi_relative else xi)
            order = np.argsort(-ei, kind="stable")
            x = None
            for i in order:  # skip candidates already sampled (after quantisation)
                c = snap(float(grid[i]))
                if all(abs(c - v) > 0.5 * quantum for v in xs):
                    x = c
                    break
            if x is None:
                x = snap(float(grid[int(order[0])]))
        y = float(objective(x))
        xs.append(x)
        ys.append(y)
        log.append((rnd, x, y, float(min(ys))))
    i = int(np.argmin(ys))
    return TuneResult(xs[i], ys[i], log)


def grid_tune(objective, lo, hi, points: int = 8, quantum: float = 1.0) -> TuneResult:
    """Search space divided into `points` equal parts; ties -> smallest S_p."""
    xs = [float(min(hi, max(quantum, math.ceil((lo + (hi - lo) * (i + 1) / points) / quantum) * quantum)))
          for i in range(points)]
    ys = [float(objective(x)) for x in xs]
    i = int(np.argmin(ys))
    return TuneResult(xs[i], ys[i], [(r, x, y, float(min(ys[:r + 1]))) for r, (x, y) in enumerate(zip(xs, ys))])


def random_tune(objective, lo, hi, draws: int = 8, seed: int = 0, quantum: float = 1.0) -> TuneResult:
    rng = np.random.default_rng(seed)
    xs = [float(min(hi, max(quantum, math.ceil((lo + (hi - lo) * rng.uniform(1e-9, 1.0)) / quantum) * quantum)))
          for _ in range(draws)]
    ys = [float(objective(x)) for x in xs]
    i = int(np.argmin(ys))
    return TuneResult(xs[i], ys[i], [(r, x, y, float(min(ys[:r + 1]))) for r, (x, y) in enumerate(zip(xs, ys))])


def retune_trigger(current: float, predicted: float, delta: float = 0.1) -> bool:
    """Eq.(18): re-run BO iff |T − F̂(S_p*)| / F̂(S_p*) > δ."""
    if predicted <= 0 or delta <= 0:
        raise ValueError("predicted and delta must be positive")
    return abs(current - predicted) / predicted > delta
