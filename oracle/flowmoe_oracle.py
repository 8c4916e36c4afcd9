"""FlowMoE block oracle — plain, slow, fp64.  TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this module.  The product path
(``paper_2510_00207_b200``) never imports it and shares no code with it; the
only shared module is ``synth`` (seeded inputs, no method arithmetic).

What it computes (paper = /root/reference/PAPER.md, "P:n"):
one transformer-MoE block — MHA, gating softmax + top-k,
capacity C = f·k·B·N/E (ceil per SPEC S:61), dispatch A2A to the
experts, expert FFN M×H then H×M, combine A2A —
forward and backward, for P simulated workers with experts sharded
contiguously (expert parallelism) and the replicated MHA+gate gradients
summed by all-reduce.  FlowMoE "only changes the scheduling order"
(Eqs.(19)-(23) P:1175-1202): the R-chunk pipelined block has exactly the
unchunked block's result, so this is the plain definition evaluated directly.
The chunk index matters only through the per-chunk capacity (reading Q2).

Readings of silent/garbled points:
Q1 chunks are whole sequences, or (Q1', causal only) contiguous slices of one
sequence when R exceeds the number of sequences — chunked prefill, whose
attention result is the causal attention's, so only the per-chunk capacity
depends on the chunking; Q2 capacity ceil per (worker, chunk);
Q3 slot-major-then-token position order, drop if pos >= C, f=0 dropless;
Q4 top-k on logits, ties -> lower expert index; Q5 renormalised top-k weights
for k>=2, raw softmax prob for k=1; Q6 gate has no bias; Q7 MHA has no biases,
scale 1/sqrt(d_h), optional causal mask and residual; Q8 experts have b1,b2
and GELU(erf); Q9 AR = sum of fp32 grads; Q12 rank p owns experts
[p·E/P, (p+1)·E/P).

Pins (tests/test_oracle_*.py): brute-force top-k, softmax closed forms,
SPEC capacity/partition examples, route invariants + sequential brute force,
dispatch∘combine identity, attention special cases, identity-expert closed
form, central finite differences for every gradient, chunked == unchunked,
P-worker == single workers, chunked AR == whole sum, 4M²+ME sizes.
"Block output values" beyond those are parity-unpinned (the paper prints no
numeric block outputs).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
from scipy.special import erf as _erf  # library primitive: the error function

# ---------------------------------------------------------------------------
# scalar pieces
# ---------------------------------------------------------------------------


def capacity(f: float, k: int, T_r: int, E: int) -> int:
    """C = f·k·B·N/E, rounded up (reading Q2).

    ``f`` is taken as its float32 value (the C-ABI field is a float) and the
    product is formed in double in the order f·k·T_r/E.  f = 0 means dropless
    (C = T_r: a token picks an expert at most once, so load <= T_r).
    """
    if f == 0:
        return int(T_r)
    return int(math.ceil(float(np.float32(f)) * k * T_r / E))


def partition_ar(nbytes: int, s_p: int) -> list[int]:
    """Alg. 2 PARTITION: floor(bytes/S_p) chunks of S_p plus a
    remainder chunk."""
    if nbytes <= 0 or s_p <= 0:
        raise ValueError("partition_ar needs positive sizes")
    n_full, rem = divmod(nbytes, s_p)
    return [s_p] * n_full + ([rem] if rem else [])


def ar_param_count(M: int, E: int) -> int:
    """Parameters of MHA + linear gate per block: 4M² + M·E."""
    return 4 * M * M + M * E


def expert_param_count(M: int, F: int) -> int:
    """Parameters of one expert: W1 [M×H], b1 [H], W2 [H×M], b2 [M] (reading Q8)."""
    return 2 * M * F + F + M


def gelu(z: np.ndarray) -> np.ndarray:
    """GELU_erf(z) = ½ z (1 + erf(z/√2))  (reading Q8)."""
    return 0.5 * z * (1.0 + _erf(z / math.sqrt(2.0)))


def gelu_grad(z: np.ndarray) -> np.ndarray:
    """GELU'(z) = ½(1 + erf(z/√2)) + z·exp(−z²/2)/√(2π)."""
    return 0.5 * (1.0 + _erf(z / math.sqrt(2.0))) + z * np.exp(-0.5 * z * z) / math.sqrt(2.0 * math.pi)


def softmax_rows(l: np.ndarray) -> np.ndarray:
    """Row softmax p = exp(l − max) / Σ exp(l − max)  (the gate's "softmax layer")."""
    m = l.max(axis=1, keepdims=True)
    e = np.exp(l - m)
    return e / e.sum(axis=1, keepdims=True)


# ---------------------------------------------------------------------------
# gating / routing (readings Q3-Q5)
# ---------------------------------------------------------------------------


def topk_select(logits: np.ndarray, k: int) -> np.ndarray:
    """Top-k experts per row on the logits: the k largest, ties to the smaller
    index, slot 0 the largest.  A stable sort on (−logit, index)."""
    T, E = logits.shape
    idx = np.empty((T, k), dtype=np.int32)
    for t in range(T):
        order = sorted(range(E), key=lambda e: (-float(logits[t, e]), e))
        idx[t] = order[:k]
    return idx


def gate_weights(logits: np.ndarray, idx: np.ndarray) -> np.ndarray:
    """w_j = p_{e_j} / Σ_j' p_{e_j'} for k >= 2, w_0 = p_{e_0} for k = 1 (reading Q5)."""
    p = softmax_rows(logits)
    sel = np.take_along_axis(p, idx.astype(np.int64), axis=1)
    if idx.shape[1] == 1:
        return sel
    return sel / sel.sum(axis=1, keepdims=True)


def route_positions(idx: np.ndarray, E: int, C: int):
    """Positions inside one chunk, slot-major then token order (reading Q3):
    ``for j in 0..k-1: for t in chunk: pos = cnt[e_tj]++; kept = pos < C``.
    Returns pos [T,k] int32, kept [T,k] bool, counts [E] int32 (loads before drop)."""
    T, k = idx.shape
    cnt = np.zeros(E, dtype=np.int64)
    pos = np.zeros((T, k), dtype=np.int32)
    for j in range(k):
        for t in range(T):
            e = int(idx[t, j])
            pos[t, j] = cnt[e]
            cnt[e] += 1
    kept = pos < C
    return pos, kept, cnt.astype(np.int32)


# ---------------------------------------------------------------------------
# MHA (reading Q7)
# ---------------------------------------------------------------------------


def mha_forward(x, wqkv, wo, seq_len, n_heads, causal, residual):
    """Q,K,V = X·Wq,Wk,Wv (column blocks of Wqkv [M×3M]); per sequence and head
    ctx = softmax(QKᵀ/√d_h [+causal mask])·V; A = ctx·Wo (+X if residual)."""
    T, M = x.shape
    dh = M // n_heads
    qkv = x @ wqkv
    q, k, v = qkv[:, :M], qkv[:, M:2 * M], qkv[:, 2 * M:]
    ctx = np.zeros((T, M))
    probs = {}
    for s in range(T // seq_len):
        rows = slice(s * seq_len, (s + 1) * seq_len)
        for h in range(n_heads):
            cols = slice(h * dh, (h + 1) * dh)
            sc = q[rows, cols] @ k[rows, cols].T / math.sqrt(dh)
            if causal:
                sc = np.where(np.tril(np.ones((seq_len, seq_len), dtype=bool)), sc, -np.inf)
            pm = np.exp(sc - sc.max(axis=1, keepdims=True))
            pm = pm / pm.sum(axis=1, keepdims=True)
            probs[(s, h)] = pm
            ctx[rows, cols] = pm @ v[rows, cols]
    a = ctx @ wo
    if residual:
        a = a + x
    cache = dict(x=x, q=q, k=k, v=v, ctx=ctx, probs=probs)
    return a, cache


def mha_backward(d_a, cache, wqkv, wo, seq_len, n_heads, residual):
    """Reverse mode of mha_forward:
    dctx = dA·Woᵀ, dWo = ctxᵀ·dA; dV = Pᵀ·dctx; dP = dctx·Vᵀ;
    dS = P⊙(dP − rowsum(dP⊙P)); dQ = dS·K/√d_h; dK = dSᵀ·Q/√d_h;
    dX = dQKV·Wqkvᵀ (+dA if residual); dWqkv = Xᵀ·dQKV."""
    x, q, k, v, ctx = cache["x"], cache["q"], cache["k"], cache["v"], cache["ctx"]
    T, M = x.shape
    dh = M // n_heads
    d_wo = ctx.T @ d_a
    d_ctx = d_a @ wo.T
    dq = np.zeros_like(q)
    dk = np.zeros_like(k)
    dv = np.zeros_like(v)
    for s in range(T // seq_len):
        rows = slice(s * seq_len, (s + 1) * seq_len)
        for h in range(n_heads):
            cols = slice(h * dh, (h + 1) * dh)
            pm = cache["probs"][(s, h)]
            dc = d_ctx[rows, cols]
            dv[rows, cols] = pm.T @ dc
            dp = dc @ v[rows, cols].T
            ds = pm * (dp - (dp * pm).sum(axis=1, keepdims=True))
            dq[rows, cols] = ds @ k[rows, cols] / math.sqrt(dh)
            dk[rows, cols] = ds.T @ q[rows, cols] / math.sqrt(dh)
    d_qkv = np.concatenate([dq, dk, dv], axis=1)
    d_wqkv = x.T @ d_qkv
    d_x = d_qkv @ wqkv.T
    if residual:
        d_x = d_x + d_a
    return d_x, d_wqkv, d_wo


# ---------------------------------------------------------------------------
# experts (reading Q8)
# ---------------------------------------------------------------------------


def expert_forward(rows, w1, b1, w2, b2):
    """Z = x·W1 + b1; H = GELU(Z); Y = H·W2 + b2."""
    z = rows @ w1 + b1
    h = gelu(z)
    return h @ w2 + b2, z, h


def expert_backward(d_y, rows, z, h, w1, w2):
    """dZ = (dY·W2ᵀ)⊙GELU'(Z); dW2 = Hᵀ·dY; db2 = Σ dY; dW1 = xᵀ·dZ; db1 = Σ dZ; dx = dZ·W1ᵀ."""
    d_z = (d_y @ w2.T) * gelu_grad(z)
    return d_z @ w1.T, rows.T @ d_z, d_z.sum(axis=0), h.T @ d_y, d_y.sum(axis=0)


# ---------------------------------------------------------------------------
# the block, P simulated workers
# ---------------------------------------------------------------------------


@dataclass
class Routing:
    idx: np.ndarray      # [T,k] int32 expert ids
    w: np.ndarray        # [T,k] gate weights
    pos: np.ndarray      # [T,k] int32 position inside the (chunk, expert) capacity buffer
    kept: np.ndarray     # [T,k] bool
    counts: np.ndarray   # [R,E] int32 loads before the capacity drop
    logits: np.ndarray   # [T,E]


@dataclass
class BlockState:
    mha: list = field(default_factory=list)        # per worker
    a: list = field(default_factory=list)          # per worker [T,M] (I')
    route: list = field(default_factory=list)      # per worker Routing
    exp_cache: dict = field(default_factory=dict)  # e -> (src list, rows, z, h, y)


def route_worker(cfg, a, wg, forced_idx=None, logits=None):
    """Gate (logits = A·Wg), top-k, weights and per-chunk positions for one worker."""
    T_r = cfg.T // cfg.R
    if logits is None:
        logits = a @ wg
    idx = topk_select(logits, cfg.top_k) if forced_idx is None else np.asarray(forced_idx, np.int32)
    w = gate_weights(logits, idx)
    C = capacity(cfg.capacity_factor, cfg.top_k, T_r, cfg.E)
    pos = np.zeros_like(idx)
    kept = np.zeros(idx.shape, dtype=bool)
    counts = np.zeros((cfg.R, cfg.E), dtype=np.int32)
    for r in range(cfg.R):
        rs = slice(r * T_r, (r + 1) * T_r)
        pos[rs], kept[rs], counts[r] = route_positions(idx[rs], cfg.E, C)
    return Routing(idx=idx, w=w, pos=pos, kept=kept, counts=counts, logits=logits)


def block_forward(cfg, rep, xs, forced=None):
    """Forward of one block on P workers.  ``rep``: replicated weights
    (wqkv, wo, wg and all experts w1,b1,w2,b2 indexed by global e); ``xs``: list
    of P worker inputs [T,M]; ``forced``: optional list of [T,k] indices
    (forced-routing mode, §8(c.1) step 12).  Returns (ys, state)."""
    P = len(xs)
    st = BlockState()
    for p in range(P):
        a, cache = mha_forward(xs[p], rep["wqkv"], rep["wo"], cfg.seq_len, cfg.n_heads,
                               cfg.causal, cfg.residual)
        st.mha.append(cache)
        st.a.append(a)
        st.route.append(route_worker(cfg, a, rep["wg"], None if forced is None else forced[p]))
    ys = [np.zeros_like(x) for x in xs]
    for e in range(cfg.E):
        src = []
        for p in range(P):
            tt, jj = np.nonzero((st.route[p].idx == e) & st.route[p].kept)
            src += [(p, int(t), int(j)) for t, j in zip(tt, jj)]
        if not src:
            st.exp_cache[e] = (src, None, None, None, None)
            continue
        rows = np.stack([st.a[p][t] for (p, t, j) in src])
        y, z, h = expert_forward(rows, rep["w1"][e], rep["b1"][e], rep["w2"][e], rep["b2"][e])
        st.exp_cache[e] = (src, rows, z, h, y)
        for i, (p, t, j) in enumerate(src):
            ys[p][t] += st.route[p].w[t, j] * y[i]
    if cfg.residual:
        for p in range(P):
            ys[p] += st.a[p]
    return ys, st


def block_backward(cfg, rep, st, dys):
    """Exact reverse mode of block_forward (§8(c.1) step 10-11).
    Returns (dxs, grad_flat, expert_grads) where grad_flat is the all-reduced
    (summed over workers) [dWqkv | dWo | dWg] fp64 vector and expert_grads maps
    global e -> (dW1, db1, dW2, db2)."""
    P, T, k, E, M = len(dys), cfg.T, cfg.top_k, cfg.E, cfg.M
    d_as = [np.zeros((T, M)) for _ in range(P)]
    d_w = [np.zeros((T, k)) for _ in range(P)]
    exp_grads = {}
    for e in range(E):
        src, rows, z, h, y = st.exp_cache[e]
        if not src:
            exp_grads[e] = (np.zeros((M, cfg.d_ffn)), np.zeros(cfg.d_ffn),
                            np.zeros((cfg.d_ffn, M)), np.zeros(M))
            continue
        d_y = np.stack([st.route[p].w[t, j] * dys[p][t] for (p, t, j) in src])
        for i, (p, t, j) in enumerate(src):
            d_w[p][t, j] = float(dys[p][t] @ y[i])
        d_rows, dw1, db1, dw2, db2 = expert_backward(d_y, rows, z, h, rep["w1"][e], rep["w2"][e])
        exp_grads[e] = (dw1, db1, dw2, db2)
        for i, (p, t, j) in enumerate(src):
            d_as[p][t] += d_rows[i]
    dxs = []
    d_wqkv = np.zeros((M, 3 * M))
    d_wo = np.zeros((M, M))
    d_wg = np.zeros((M, E))
    for p in range(P):
        ro = st.route[p]
        d_l = gate_logits_grad(ro.logits, ro.idx, ro.w, d_w[p])
        d_a = d_as[p] + d_l @ rep["wg"].T
        if cfg.residual:
            d_a = d_a + dys[p]
        d_wg += st.a[p].T @ d_l
        d_x, dwqkv_p, dwo_p = mha_backward(d_a, st.mha[p], rep["wqkv"], rep["wo"], cfg.seq_len,
                                           cfg.n_heads, cfg.residual)
        d_wqkv += dwqkv_p
        d_wo += dwo_p
        dxs.append(d_x)
    grad_flat = np.concatenate([d_wqkv.ravel(), d_wo.ravel(), d_wg.ravel()])
    return dxs, grad_flat, exp_grads


def gate_logits_grad(logits, idx, w, d_w):
    """dℓ from dw (reading Q5).  k >= 2: on the selected set
    dℓ_{e_j} = w_j (dw_j − Σ_j' w_j' dw_j'), 0 elsewhere.
    k = 1: dℓ_e = p_e (g_e − Σ_e' p_e' g_e') with g_{e_0} = dw_0, other g = 0."""
    T, E = logits.shape
    k = idx.shape[1]
    d_l = np.zeros((T, E))
    if k == 1:
        p = softmax_rows(logits)
        g = np.zeros((T, E))
        g[np.arange(T), idx[:, 0]] = d_w[:, 0]
        d_l = p * (g - (p * g).sum(axis=1, keepdims=True))
    else:
        inner = (w * d_w).sum(axis=1, keepdims=True)
        vals = w * (d_w - inner)
        for j in range(k):
            d_l[np.arange(T), idx[:, j]] += vals[:, j]
    return d_l


# ---------------------------------------------------------------------------
# explicit expert-parallel data movement: send buffers,
# simulated A2A, capacity-padded expert inputs, combine.
# ---------------------------------------------------------------------------


def dispatch_buffers(cfg, a, route, r):
    """send_p[e][pos] = A[t] for kept slots of chunk r; padding rows are zero.
    Shape [E, C, M] (G(I') ∈ R^{E×C×M})."""
    T_r = cfg.T // cfg.R
    C = capacity(cfg.capacity_factor, cfg.top_k, T_r, cfg.E)
    send = np.zeros((cfg.E, C, cfg.M))
    for t in range(r * T_r, (r + 1) * T_r):
        for j in range(cfg.top_k):
            if route.kept[t, j]:
                send[route.idx[t, j], route.pos[t, j]] = a[t]
    return send


def alltoall(sends, P):
    """Simulated A2A: recv_q[p][e_l] = send_p[q·E/P + e_l] (experts contiguous per rank, Q12)."""
    E = sends[0].shape[0]
    El = E // P
    return [np.stack([sends[p][q * El:(q + 1) * El] for p in range(P)]) for q in range(P)]


def combine_from_buffers(cfg, route, r, ybuf):
    """out[t] = Σ_{kept j} w_j · Y[e_j][pos_j] over chunk r (dropped slots add 0)."""
    T_r = cfg.T // cfg.R
    out = np.zeros((T_r, ybuf.shape[-1]))
    for i, t in enumerate(range(r * T_r, (r + 1) * T_r)):
        for j in range(cfg.top_k):
            if route.kept[t, j]:
                out[i] += route.w[t, j] * ybuf[route.idx[t, j], route.pos[t, j]]
    return out


def block_forward_ep(cfg, rep, xs, forced=None):
    """The same forward computed the expert-parallel way, chunk by chunk:
    AT_r -> D_r (A2A) -> E_r on the owner -> C_r (A2A) -> merge (Eqs.(3)-(4))."""
    P = len(xs)
    El = cfg.E // P
    T_r = cfg.T // cfg.R
    a_s, routes = [], []
    for p in range(P):
        a, _ = mha_forward(xs[p], rep["wqkv"], rep["wo"], cfg.seq_len, cfg.n_heads, cfg.causal,
                           cfg.residual)
        a_s.append(a)
        routes.append(route_worker(cfg, a, rep["wg"], None if forced is None else forced[p]))
    ys = [np.zeros_like(x) for x in xs]
    for r in range(cfg.R):
        sends = [dispatch_buffers(cfg, a_s[p], routes[p], r) for p in range(P)]
        recvs = alltoall(sends, P)          # recv_q [P(src)][El][C][M]
        outs = []
        for q in range(P):
            yq = np.zeros_like(recvs[q])
            for el in range(El):
                e = q * El + el
                for p in range(P):
                    yq[p, el], _, _ = expert_forward(recvs[q][p, el], rep["w1"][e], rep["b1"][e],
                                                     rep["w2"][e], rep["b2"][e])
            outs.append(yq)
        # combine A2A: worker p gets back [E][C][M] with e = q·El + el
        for p in range(P):
            ybuf = np.concatenate([outs[q][p] for q in range(P)], axis=0)
            ys[p][r * T_r:(r + 1) * T_r] = combine_from_buffers(cfg, routes[p], r, ybuf)
    if cfg.residual:
        for p in range(P):
            ys[p] += a_s[p]
    return ys


# ---------------------------------------------------------------------------
# chunked all-reduce (Alg. 2)
# ---------------------------------------------------------------------------


def allreduce_chunked(bufs, chunk_elems, dtype=np.float32):
    """Sum over workers, chunk by chunk in flat-buffer order (reading Q11).
    Each chunk's sum is formed in ``dtype`` in worker order 0..P−1."""
    n = bufs[0].size
    out = np.zeros(n, dtype=dtype)
    for start in range(0, n, chunk_elems):
        end = min(n, start + chunk_elems)
        acc = np.zeros(end - start, dtype=dtype)
        for b in bufs:
            acc = (acc + b[start:end].astype(dtype)).astype(dtype)
        out[start:end] = acc
    return out

