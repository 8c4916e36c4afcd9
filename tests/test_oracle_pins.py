"""Pins of the CPU oracle against what the paper and mathematics fix (no GPU).

Each test pins a part of oracle/flowmoe_oracle.py to something other than
itself: printed values (tests/golden/paper_values.json, cited), closed forms,
brute force on tiny inputs, invariants, and finite differences.
"""
import itertools
import json
import math
import os

import numpy as np
import pytest

import oracle as o
from synth import BlockConfig, PRESETS, gen_replicated, gen_worker

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))


# --------------------------------------------------------------- printed values
def test_capacity_spec_examples():
    for ex in GOLDEN["capacity"]:
        assert o.capacity(ex["f"], ex["k"], ex["tokens"], ex["E"]) == ex["C"], ex["cite"]
    assert o.capacity(0.0, 2, 256, 4) == 256  # dropless reading (Q3)


def test_partition_ar_spec_examples():
    for ex in GOLDEN["partition_ar"]:
        assert o.partition_ar(ex["bytes"], ex["S_p"]) == ex["chunks"], ex["cite"]
    with pytest.raises(ValueError):
        o.partition_ar(0, 4)


def test_ar_param_count_spec_examples():
    for ex in GOLDEN["ar_params"]:
        assert o.ar_param_count(ex["M"], ex["E"]) == ex["params"], ex["cite"]
        if "bytes_fp32" in ex:
            assert 4 * o.ar_param_count(ex["M"], ex["E"]) == ex["bytes_fp32"]


def test_table3_expert_counts_need_biases():
    """Table 3's expert parameter counts are reproduced (to the printed 0.1M)
    only with b1, b2 present (reading Q8); without biases they miss."""
    rows = GOLDEN["table3"]["rows"]
    misses_without_bias = 0
    for r in rows:
        E = r["E_per_P"] * 16
        with_b = o.expert_param_count(r["M"], r["H"]) * E * r["L"] / 1e6
        no_b = 2 * r["M"] * r["H"] * E * r["L"] / 1e6
        assert abs(with_b - r["experts_M"]) <= 0.1 + 1e-9, r["model"]
        misses_without_bias += abs(no_b - r["experts_M"]) > 0.1
    assert misses_without_bias >= len(rows) - 1  # GPT2-Tiny is too small to tell (0.07M)


# --------------------------------------------------------------- gating
def _brute_topk(l, k):
    E = len(l)
    key = [(float(l[e]), -e) for e in range(E)]
    found = []
    for S in itertools.combinations(range(E), k):
        rest = [e for e in range(E) if e not in S]
        if not rest or min(key[e] for e in S) > max(key[e] for e in rest):
            found.append(sorted(S, key=lambda e: key[e], reverse=True))
    assert len(found) == 1
    return found[0]


@pytest.mark.parametrize("E,k", [(4, 1), (4, 2), (6, 3), (8, 2), (8, 8)])
def test_topk_bruteforce_random_and_ties(E, k):
    rng = np.random.default_rng(E * 10 + k)
    cases = [rng.standard_normal(E) for _ in range(30)]
    cases += [np.round(rng.standard_normal(E) * 2) / 2 for _ in range(30)]  # many ties
    cases += [np.zeros(E), np.arange(E)[::-1].astype(float), np.array([1.0] * E)]
    L = np.stack(cases)
    idx = o.topk_select(L, k)
    for t in range(L.shape[0]):
        assert list(idx[t]) == _brute_topk(L[t], k)
        # library check: stable argsort on the negated logits
        assert list(idx[t]) == list(np.argsort(-L[t], kind="stable")[:k])


def test_gate_weights_closed_forms():
    rng = np.random.default_rng(1)
    l = rng.standard_normal((50, 8))
    p = o.softmax_rows(l)
    assert np.allclose(p.sum(1), 1.0, atol=1e-15, rtol=0)
    # two-way softmax = logistic sigmoid of the logit difference
    l2 = l[:, :2]
    assert np.allclose(o.softmax_rows(l2)[:, 0], 1.0 / (1.0 + np.exp(l2[:, 1] - l2[:, 0])), rtol=1e-14)
    idx2 = o.topk_select(l, 2)
    w2 = o.gate_weights(l, idx2)
    assert np.allclose(w2.sum(1), 1.0, atol=1e-15, rtol=0)
    d = l[np.arange(50), idx2[:, 1]] - l[np.arange(50), idx2[:, 0]]
    assert np.allclose(w2[:, 0], 1.0 / (1.0 + np.exp(d)), rtol=1e-14)
    idx1 = o.topk_select(l, 1)
    w1 = o.gate_weights(l, idx1)
    assert np.allclose(w1[:, 0], np.exp(l).max(1) / np.exp(l).sum(1), rtol=1e-14)


# --------------------------------------------------------------- routing
def _brute_positions(idx, E, C):
    T, k = idx.shape
    pos = np.zeros((T, k), dtype=np.int64)
    for t in range(T):
        for j in range(k):
            pos[t, j] = sum(1 for j2 in range(k) for t2 in range(T)
                            if idx[t2, j2] == idx[t, j] and (j2, t2) < (j, t))
    return pos


@pytest.mark.parametrize("T,E,k,C", [(16, 4, 2, 5), (12, 8, 3, 2), (20, 4, 1, 3), (9, 3, 3, 9)])
def test_route_positions_bruteforce_and_invariants(T, E, k, C):
    rng = np.random.default_rng(T + E + k)
    idx = np.stack([rng.permutation(E)[:k] for _ in range(T)]).astype(np.int32)
    pos, kept, counts = o.route_positions(idx, E, C)
    assert np.array_equal(pos, _brute_positions(idx, E, C))
    assert np.array_equal(kept, pos < C)
    for e in range(E):
        sel = (idx == e)
        assert counts[e] == sel.sum()
        assert sorted(pos[sel & kept].tolist()) == list(range(min(counts[e], C)))
    assert kept.sum() == sum(min(int(c), C) for c in counts)
    pairs = {(int(idx[t, j]), int(pos[t, j])) for t in range(T) for j in range(k) if kept[t, j]}
    assert len(pairs) == kept.sum()  # (e, pos) -> (t, j) injective


def test_first_choices_outrank_second_choices():
    """Slot-major order (Q3): a kept 2nd choice never displaces a 1st choice."""
    idx = np.array([[0, 1]] * 3 + [[1, 0]] * 3, dtype=np.int32)
    pos, kept, _ = o.route_positions(idx, 2, 3)
    assert kept[:, 0].all() and not kept[:, 1].any()


# --------------------------------------------------------------- data movement
def test_dispatch_combine_identity_bitexact():
    """k=1, w=1, identity expert, dropless: combine(dispatch(A)) == A bit-exact,
    and the dispatch is a bijection of tokens onto kept slots."""
    cfg = BlockConfig(T=32, seq_len=8, M=16, n_heads=2, E=4, top_k=1, d_ffn=8, R=2,
                      capacity_factor=0.0, dtype="f32")
    rng = np.random.default_rng(3)
    a = rng.standard_normal((cfg.T, cfg.M))
    route = o.route_worker(cfg, a, rng.standard_normal((cfg.M, cfg.E)))
    route.w[:] = 1.0
    for r in range(cfg.R):
        send = o.dispatch_buffers(cfg, a, route, r)
        out = o.combine_from_buffers(cfg, route, r, send)
        assert np.array_equal(out, a[r * 16:(r + 1) * 16])
        nz = np.abs(send).sum(-1) != 0
        assert nz.sum() == 16


def test_alltoall_is_transpose():
    P, El, C, M = 3, 2, 2, 1
    sends = [np.arange(P * El * C * M).reshape(P * El, C, M) + 100 * p for p in range(P)]
    recvs = o.alltoall(sends, P)
    for q in range(P):
        for p in range(P):
            for el in range(El):
                assert np.array_equal(recvs[q][p, el], sends[p][q * El + el])


# --------------------------------------------------------------- attention
def _mha(x, wqkv, wo, N, h, causal):
    return o.mha_forward(x, wqkv, wo, N, h, causal, 0)[1]["ctx"]


def test_attention_special_cases():
    rng = np.random.default_rng(5)
    M, h = 8, 2
    x = rng.standard_normal((12, M))
    wqkv = rng.standard_normal((M, 3 * M))
    wo = np.eye(M)
    v = x @ wqkv[:, 2 * M:]
    # N = 1 -> ctx = V
    assert np.allclose(_mha(x, wqkv, wo, 1, h, 0), v, rtol=1e-14, atol=1e-14)
    # Q = 0 -> equal scores -> mean of V over the sequence (causal: prefix mean)
    wz = wqkv.copy()
    wz[:, :M] = 0
    ctx = _mha(x, wz, wo, 4, h, 0)
    for s in range(3):
        assert np.allclose(ctx[4 * s:4 * s + 4], v[4 * s:4 * s + 4].mean(0), rtol=1e-13)
    ctx = _mha(x, wz, wo, 4, h, 1)
    for s in range(3):
        for i in range(4):
            assert np.allclose(ctx[4 * s + i], v[4 * s:4 * s + i + 1].mean(0), rtol=1e-13)
    # causal first row of every sequence is V_0 for any Q, K
    ctx = _mha(x, wqkv, wo, 4, h, 1)
    assert np.allclose(ctx[::4], v[::4], rtol=1e-13)


def test_attention_heads_are_independent_textbook():
    """Each head equals the textbook single-head softmax(QKᵀ/√d)V computed with
    scipy.special.softmax on that head's columns."""
    from scipy.special import softmax
    rng = np.random.default_rng(6)
    M, h, N = 8, 2, 5
    x = rng.standard_normal((N, M))
    wqkv = rng.standard_normal((M, 3 * M))
    ctx = _mha(x, wqkv, np.eye(M), N, h, 0)
    q, k, v = x @ wqkv[:, :M], x @ wqkv[:, M:2 * M], x @ wqkv[:, 2 * M:]
    for hh in range(h):
        c = slice(4 * hh, 4 * hh + 4)
        ref = softmax(q[:, c] @ k[:, c].T / 2.0, axis=1) @ v[:, c]
        assert np.allclose(ctx[:, c], ref, rtol=1e-13)


# --------------------------------------------------------------- experts
def test_gelu_closed_form_and_identity_expert():
    z = np.linspace(-6, 6, 101)
    # GELU(z) − GELU(−z) = z exactly in real arithmetic
    assert np.allclose(o.gelu(z) - o.gelu(-z), z, atol=1e-14)
    assert o.gelu(np.array([0.0]))[0] == 0.0
    # GELU'(0) = 1/2 and finite differences elsewhere
    assert abs(o.gelu_grad(np.array([0.0]))[0] - 0.5) < 1e-15
    hh = 1e-6
    fd = (o.gelu(z + hh) - o.gelu(z - hh)) / (2 * hh)
    assert np.allclose(fd, o.gelu_grad(z), atol=1e-8)
    # value pins (the odd-part identities above also hold for tanh-GELU and for erf
    # without the 1/√2): GELU(z) = z·Φ(z) with Φ the standard normal CDF (reading Q8),
    # Φ(1) = 0.8413447460685429 and φ(1) = e^{-1/2}/√(2π) = 0.24197072451914337
    # (normal-distribution tables, Abramowitz & Stegun 26.2), so GELU(1) = Φ(1),
    # GELU(-1) = -(1 - Φ(1)), GELU'(1) = Φ(1) + φ(1), GELU'(-1) = 1 - Φ(1) - φ(1).
    phi1, dens1 = 0.8413447460685429, 0.24197072451914337
    g = o.gelu(np.array([1.0, -1.0, 2.0]))
    assert abs(g[0] - phi1) < 1e-15
    assert abs(g[1] + (1.0 - phi1)) < 1e-15
    assert abs(g[2] - 2.0 * 0.9772498680518208) < 1e-14  # Φ(2) = 0.9772498680518208
    gg = o.gelu_grad(np.array([1.0, -1.0]))
    assert abs(gg[0] - (phi1 + dens1)) < 1e-15
    assert abs(gg[1] - (1.0 - phi1 - dens1)) < 1e-15
    # and against an independent library CDF over the whole range
    from scipy.special import ndtr
    assert np.allclose(o.gelu(z), z * ndtr(z), rtol=1e-14, atol=1e-15)
    # identity expert: W1 = [I, −I], W2 = [I; −I], b = 0  ->  FFN(x) = x
    M = 6
    w1 = np.concatenate([np.eye(M), -np.eye(M)], axis=1)
    w2 = np.concatenate([np.eye(M), -np.eye(M)], axis=0)
    x = np.random.default_rng(7).standard_normal((9, M))
    y, _, _ = o.expert_forward(x, w1, np.zeros(2 * M), w2, np.zeros(M))
    assert np.allclose(y, x, atol=1e-14)


def test_block_with_identity_experts_returns_attention_output():
    """With identity experts, dropless, k>=2 (Σw=1): MoE output = A (I')."""
    cfg = BlockConfig(T=16, seq_len=4, M=8, n_heads=2, E=4, top_k=2, d_ffn=16, R=2,
                      capacity_factor=0.0, dtype="f32", P=2)
    rep = gen_replicated(cfg)
    M = cfg.M
    rep["w1"] = np.stack([np.concatenate([np.eye(M), -np.eye(M)], axis=1)] * cfg.E)
    rep["w2"] = np.stack([np.concatenate([np.eye(M), -np.eye(M)], axis=0)] * cfg.E)
    rep["b1"][:] = 0
    rep["b2"][:] = 0
    xs = [gen_worker(cfg, p)["x"] for p in range(2)]
    ys, st = o.block_forward(cfg, rep, xs)
    for p in range(2):
        assert np.allclose(ys[p], st.a[p], atol=1e-13)
    ys_ep = o.block_forward_ep(cfg, rep, xs)
    for p in range(2):
        assert np.allclose(ys_ep[p], st.a[p], atol=1e-13)


# --------------------------------------------------------------- whole block
TINY = BlockConfig(T=8, seq_len=4, M=8, n_heads=2, E=4, top_k=2, d_ffn=16, R=2,
                   capacity_factor=1.0, causal=0, residual=0, P=2, dtype="f32")


def _tiny_setup(cfg, seed_block=0):
    rep = gen_replicated(cfg, block=seed_block)
    ws = [gen_worker(cfg, p, block=seed_block) for p in range(cfg.P)]
    return rep, [w["x"] for w in ws], [w["dy"] for w in ws]


def _loss(cfg, rep, xs, dys, forced=None):
    ys, _ = o.block_forward(cfg, rep, xs, forced)
    return sum(float((dy * y).sum()) for dy, y in zip(dys, ys))


def _margins_ok(cfg, rep, xs):
    _, st = o.block_forward(cfg, rep, xs)
    for ro in st.route:
        s = np.sort(ro.logits, axis=1)[:, ::-1]
        k = cfg.top_k
        if k < cfg.E and np.min(s[:, k - 1] - s[:, k]) < 1e-3:
            return False
    return True


@pytest.mark.parametrize("causal,residual,k,f", [(0, 0, 2, 1.0), (1, 1, 2, 1.0), (0, 1, 1, 0.0),
                                                 (1, 0, 3, 1.0)])
def test_block_gradients_finite_differences(causal, residual, k, f):
    cfg = TINY.replace(causal=causal, residual=residual, top_k=k, capacity_factor=f)
    rep, xs, dys = _tiny_setup(cfg, seed_block=k + 3 * causal)
    assert _margins_ok(cfg, rep, xs)
    ys, st = o.block_forward(cfg, rep, xs)
    if f == 1.0:
        assert any((~ro.kept).any() for ro in st.route), "want capacity drops in the case"
    dxs, gflat, eg = o.block_backward(cfg, rep, st, dys)
    M, E = cfg.M, cfg.E
    nq = 3 * M * M
    analytic = {
        "wqkv": gflat[:M * 3 * M].reshape(M, 3 * M),
        "wo": gflat[M * 3 * M:M * 3 * M + M * M].reshape(M, M),
        "wg": gflat[4 * M * M:].reshape(M, E),
        "w1": np.stack([eg[e][0] for e in range(E)]),
        "b1": np.stack([eg[e][1] for e in range(E)]),
        "w2": np.stack([eg[e][2] for e in range(E)]),
        "b2": np.stack([eg[e][3] for e in range(E)]),
    }
    assert gflat.size == o.ar_param_count(M, E) and nq == 3 * M * M
    rng = np.random.default_rng(11)
    worst = 0.0
    for name, g in analytic.items():
        flat = rep[name].reshape(-1)
        for i in rng.choice(flat.size, size=min(flat.size, 24), replace=False):
            hh = 1e-6 * max(1.0, abs(flat[i]))
            old = flat[i]
            flat[i] = old + hh
            lp = _loss(cfg, rep, xs, dys)
            flat[i] = old - hh
            lm = _loss(cfg, rep, xs, dys)
            flat[i] = old
            fd = (lp - lm) / (2 * hh)
            worst = max(worst, abs(fd - g.reshape(-1)[i]) / max(1.0, np.abs(g).max()))
    for p in range(cfg.P):
        flat = xs[p].reshape(-1)
        for i in rng.choice(flat.size, size=24, replace=False):
            hh = 1e-6 * max(1.0, abs(flat[i]))
            old = flat[i]
            flat[i] = old + hh
            lp = _loss(cfg, rep, xs, dys)
            flat[i] = old - hh
            lm = _loss(cfg, rep, xs, dys)
            flat[i] = old
            worst = max(worst, abs((lp - lm) / (2 * hh) - dxs[p].reshape(-1)[i])
                        / max(1.0, np.abs(dxs[p]).max()))
    assert worst < 1e-6, worst


def test_forced_routing_gradients_finite_differences():
    cfg = TINY.replace(residual=1)
    rep, xs, dys = _tiny_setup(cfg, seed_block=9)
    forced = [gen_worker(cfg, p, block=9)["forced_idx"] for p in range(cfg.P)]
    ys, st = o.block_forward(cfg, rep, xs, forced)
    _, gflat, _ = o.block_backward(cfg, rep, st, dys)
    flat = rep["wg"].reshape(-1)
    g = gflat[4 * cfg.M * cfg.M:]
    for i in range(flat.size):
        old = flat[i]
        flat[i] = old + 1e-6
        lp = _loss(cfg, rep, xs, dys, forced)
        flat[i] = old - 1e-6
        lm = _loss(cfg, rep, xs, dys, forced)
        flat[i] = old
        assert abs((lp - lm) / 2e-6 - g[i]) < 1e-7 * max(1.0, np.abs(g).max())


def test_chunked_equals_unchunked_dropless():
    """Eqs.(19)-(23)/P:520: pipelining changes only the order — R=1 and
    R in {2,4} agree (dropless, so capacity cannot differ per chunk); so do the token
    chunks R in {8,16} (2 or 1 tokens of a 4-token causal sequence per chunk, reading
    Q1': chunked prefill, Table 5's R=8 at B=4)."""
    base = BlockConfig(T=16, seq_len=4, M=8, n_heads=2, E=4, top_k=2, d_ffn=16, R=1,
                       capacity_factor=0.0, causal=1, residual=1, P=2, dtype="f32")
    rep, xs, dys = _tiny_setup(base)
    ref_y, st = o.block_forward(base, rep, xs)
    ref = o.block_backward(base, rep, st, dys)
    for R in (2, 4, 8, 16):
        cfg = base.replace(R=R)
        ys, st2 = o.block_forward(cfg, rep, xs)
        got = o.block_backward(cfg, rep, st2, dys)
        for a, b in zip(ys, ref_y):
            assert np.max(np.abs(a - b)) <= 1e-12 * np.max(np.abs(b))
        assert np.max(np.abs(got[1] - ref[1])) <= 1e-12 * np.max(np.abs(ref[1]))
        for e in range(base.E):
            for a, b in zip(got[2][e], ref[2][e]):
                assert np.max(np.abs(a - b)) <= 1e-12 * max(1e-30, np.max(np.abs(b)))
        ys_ep = o.block_forward_ep(cfg, rep, xs)
        for a, b in zip(ys_ep, ref_y):
            assert np.max(np.abs(a - b)) <= 1e-12 * np.max(np.abs(b))


def test_chunked_prefill_attention_is_causal_attention():
    """Reading Q1' (token chunks): chunk [p0, p0+n) of a causal sequence attends to the
    keys [0, p0+n) it has seen so far — brute force per query row, chunk by chunk,
    built only from the rows the chunk may read, equals the oracle's causal MHA rows."""
    rng = np.random.default_rng(7)
    N, M, h = 12, 8, 2
    dh = M // h
    x = rng.standard_normal((N, M))
    wqkv, wo = rng.standard_normal((M, 3 * M)) / np.sqrt(M), rng.standard_normal((M, M)) / np.sqrt(M)
    a_ref, _ = o.mha_forward(x, wqkv, wo, N, h, causal=1, residual=0)
    for n in (1, 3, 4, 6):
        ctx = np.zeros((N, M))
        for p0 in range(0, N, n):
            seen = x[:p0 + n] @ wqkv  # projections of the rows up to the chunk end only
            for i in range(p0, p0 + n):
                for hh in range(h):
                    q = seen[i, hh * dh:(hh + 1) * dh]
                    ks = seen[:i + 1, M + hh * dh:M + (hh + 1) * dh]
                    vs = seen[:i + 1, 2 * M + hh * dh:2 * M + (hh + 1) * dh]
                    sc = ks @ q / np.sqrt(dh)
                    p = np.exp(sc - sc.max())
                    ctx[i, hh * dh:(hh + 1) * dh] = (p / p.sum()) @ vs
        assert np.max(np.abs(ctx @ wo - a_ref)) <= 1e-12 * np.max(np.abs(a_ref))


def test_ep_forward_matches_direct_with_drops():
    cfg = PRESETS["c1"]
    rep = gen_replicated(cfg)
    xs = [gen_worker(cfg, p)["x"] for p in range(cfg.P)]
    ys, st = o.block_forward(cfg, rep, xs)
    assert any((~ro.kept).any() for ro in st.route)
    ys_ep = o.block_forward_ep(cfg, rep, xs)
    for a, b in zip(ys_ep, ys):
        assert np.max(np.abs(a - b)) <= 1e-12 * np.max(np.abs(b))


def test_p_workers_equal_single_workers():
    """EP sharding changes only placement: the P-worker block equals each worker
    computed alone (all E experts local); replicated grads = Σ_p; expert grads =
    Σ over sources."""
    cfg = PRESETS["c1"]
    rep, xs, dys = _tiny_setup(cfg)
    ys, st = o.block_forward(cfg, rep, xs)
    dxs, gflat, eg = o.block_backward(cfg, rep, st, dys)
    one = cfg.replace(P=1)
    g_sum = np.zeros_like(gflat)
    e_sum = {e: [np.zeros_like(a) for a in eg[e]] for e in range(cfg.E)}
    for p in range(cfg.P):
        y1, st1 = o.block_forward(one, rep, [xs[p]])
        dx1, g1, eg1 = o.block_backward(one, rep, st1, [dys[p]])
        assert np.max(np.abs(y1[0] - ys[p])) <= 1e-12 * np.max(np.abs(ys[p]))
        assert np.max(np.abs(dx1[0] - dxs[p])) <= 1e-12 * np.max(np.abs(dxs[p]))
        g_sum += g1
        for e in range(cfg.E):
            for i in range(4):
                e_sum[e][i] += eg1[e][i]
    assert np.max(np.abs(g_sum - gflat)) <= 1e-12 * np.max(np.abs(gflat))
    for e in range(cfg.E):
        for i in range(4):
            assert np.max(np.abs(e_sum[e][i] - eg[e][i])) <= 1e-12 * np.max(np.abs(eg[e][i]))


# --------------------------------------------------------------- all-reduce
@pytest.mark.parametrize("n,chunk", [(1000, 7), (1000, 1000), (1000, 4096), (4096, 256), (17, 16)])
def test_chunked_allreduce_equals_whole_sum_bitexact(n, chunk):
    rng = np.random.default_rng(n + chunk)
    bufs = [rng.integers(-1024, 1025, size=n).astype(np.float32) for _ in range(4)]
    got = o.allreduce_chunked(bufs, chunk)
    whole = np.sum(np.stack(bufs).astype(np.float64), axis=0).astype(np.float32)
    assert np.array_equal(got, whole)
    sizes = o.partition_ar(n * 4, chunk * 4)
    assert sum(sizes) == n * 4 and len(sizes) == -(-n // chunk)


# --------------------------------------------------------------- micro-batch scaling
def test_microbatch_loss_scaling_identity():
    """SPEC S:392-400 / Eqs.(19)-(23): Σ_r ∇(loss_r/R) = ∇L_full; unscaled ≈ R×."""
    ex = GOLDEN["microbatch_identity"]
    B, R, d = ex["B"], ex["R"], ex["dim"]
    rng = np.random.default_rng(0)
    x, y, w = rng.standard_normal((B, d)), rng.standard_normal(B), rng.standard_normal(d)

    def grad(xs, ys):  # ∇ of mean (w·x − y)²
        return (2.0 * (xs @ w - ys)[:, None] * xs).mean(0)

    full = grad(x, y)
    b = B // R
    scaled = sum(grad(x[r * b:(r + 1) * b], y[r * b:(r + 1) * b]) / R for r in range(R))
    unscaled = sum(grad(x[r * b:(r + 1) * b], y[r * b:(r + 1) * b]) for r in range(R))
    assert np.max(np.abs(scaled - full) / np.abs(full)) <= ex["max_dev"]
    assert np.allclose(unscaled, R * full)


# --------------------------------------------------------------- optimizer (reading Q17)
def test_adamw_first_step_is_signed_lr():
    """Step 1: m̂ = g and v̂ = g² exactly, so the update is lr·g/(|g|+ε) ≈ lr·sign(g)
    (plus the decoupled decay w·lr·wd) — the closed form of the first AdamW step."""
    from oracle.optim import adamw_step
    rng = np.random.default_rng(11)
    w, g = rng.standard_normal(64), rng.standard_normal(64) + 3.0 * np.sign(rng.standard_normal(64))
    z = np.zeros(64)
    w1, m1, v1 = adamw_step(w, z, z, g, lr=1e-2, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.1, step=1)
    assert np.allclose(m1, 0.1 * g, rtol=0, atol=1e-15) and np.allclose(v1, 0.001 * g * g, rtol=1e-14)
    want = w * (1 - 1e-3) - 1e-2 * g / (np.abs(g) + 1e-8)
    assert np.max(np.abs(w1 - want)) <= 1e-14
    # lr = 0 leaves the weights alone whatever the state
    w0, _, _ = adamw_step(w, m1, v1, g, lr=0.0, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.1, step=2)
    assert np.array_equal(w0, w)


def test_adamw_constant_gradient_converges_to_signed_lr_steps():
    """A constant gradient keeps m̂ = g and v̂ = g² at every step (bias correction exact),
    so without decay every step moves w by exactly lr·g/(|g|+ε)."""
    from oracle.optim import adamw_step
    g = np.array([0.5, -2.0, 1e-3])
    w, m, v = np.zeros(3), np.zeros(3), np.zeros(3)
    for t in range(1, 6):
        w, m, v = adamw_step(w, m, v, g, lr=0.1, beta1=0.9, beta2=0.99, eps=0.0, weight_decay=0.0, step=t)
    assert np.allclose(w, -5 * 0.1 * np.sign(g), rtol=1e-12, atol=1e-12)


def test_sgd_momentum_two_steps_by_hand():
    from oracle.optim import sgd_momentum_step
    w, g1, g2 = np.array([1.0, -2.0]), np.array([0.5, 0.25]), np.array([-1.0, 1.0])
    w1, b1 = sgd_momentum_step(w, np.zeros(2), g1, lr=0.1, momentum=0.9, weight_decay=0.01, step=1)
    d1 = g1 + 0.01 * w
    assert np.allclose(b1, d1) and np.allclose(w1, w - 0.1 * d1)
    w2, b2 = sgd_momentum_step(w1, b1, g2, lr=0.1, momentum=0.9, weight_decay=0.01, step=2)
    d2 = g2 + 0.01 * w1
    assert np.allclose(b2, 0.9 * d1 + d2) and np.allclose(w2, w1 - 0.1 * (0.9 * d1 + d2))


# --------------------------------------------------------------- model edges (reading Q18)
def test_xent_uniform_logits_is_log_vocab():
    """Equal logits: every labelled token costs log V exactly, and the gradient row is
    scale·(1/V − onehot)."""
    from oracle.model import xent
    T, V = 5, 7
    labels = np.array([0, 3, -1, 6, 2])
    losses, loss, dl = xent(np.full((T, V), 0.37), labels, 0.25)
    assert np.allclose(losses[[0, 1, 3, 4]], np.log(V)) and losses[2] == 0.0
    assert np.isclose(loss, 0.25 * 4 * np.log(V))
    want = np.full(V, 0.25 / V)
    want[3] -= 0.25
    assert np.allclose(dl[1], want) and np.all(dl[2] == 0.0)


def test_xent_gradient_by_finite_differences_and_shift_invariance():
    from oracle.model import xent
    rng = np.random.default_rng(5)
    T, V, s = 3, 6, 0.5
    lg = rng.standard_normal((T, V)) * 2
    labels = np.array([4, 0, 5])
    _, loss, dl = xent(lg, labels, s)
    h = 1e-6
    for t, v in [(0, 4), (1, 2), (2, 5), (2, 0)]:
        p = lg.copy(); p[t, v] += h
        m = lg.copy(); m[t, v] -= h
        fd = (xent(p, labels, s)[1] - xent(m, labels, s)[1]) / (2 * h)
        assert abs(fd - dl[t, v]) < 1e-8
    # softmax is shift invariant per row; gradient rows sum to zero
    assert np.isclose(xent(lg + np.array([[3.0], [-7.0], [0.5]]), labels, s)[1], loss)
    assert np.allclose(dl.sum(axis=1), 0.0)


def test_xent_chunked_losses_add_to_the_full_loss():
    """Eqs.(19)-(23): R chunks with scale 1/B each sum to the full mean loss, and their
    gradient rows are the full gradient's rows."""
    from oracle.model import xent
    rng = np.random.default_rng(9)
    B, V, R = 12, 5, 4
    lg = rng.standard_normal((B, V))
    labels = rng.integers(0, V, B)
    _, full, dfull = xent(lg, labels, 1.0 / B)
    parts = [xent(lg[r * (B // R):(r + 1) * (B // R)],
                  labels[r * (B // R):(r + 1) * (B // R)], 1.0 / B) for r in range(R)]
    assert np.isclose(sum(p[1] for p in parts), full)
    assert np.allclose(np.concatenate([p[2] for p in parts]), dfull)
    # and the full loss is the plain mean of -log softmax at the label
    p = np.exp(lg) / np.exp(lg).sum(axis=1, keepdims=True)
    assert np.isclose(full, -np.mean(np.log(p[np.arange(B), labels])))


def test_embedding_gather_and_scatter_brute_force():
    from oracle.model import embed_backward, embed_forward
    rng = np.random.default_rng(2)
    V, M = 6, 4
    table = rng.standard_normal((V, M))
    ids = np.array([2, 5, 2, 0, 9, 2])  # a repeated id and an out-of-range one
    x = embed_forward(table, ids)
    assert np.array_equal(x[0], table[2]) and np.array_equal(x[1], table[5]) and np.all(x[4] == 0)
    dx = rng.standard_normal((len(ids), M))
    d = embed_backward(ids, dx, V)
    assert np.allclose(d[2], dx[0] + dx[2] + dx[5]) and np.allclose(d[0], dx[3])
    assert np.all(d[[1, 3, 4]] == 0)
    # adjoint identity <embed(table), dx> = <table, embed_backward(dx)> over in-range ids
    keep = ids < V
    assert np.isclose(np.sum(embed_forward(table, ids)[keep] * dx[keep]), np.sum(table * d))


def test_lm_head_brute_force_and_adjoints():
    from oracle.model import lm_head_backward, lm_head_forward
    rng = np.random.default_rng(4)
    T, M, V = 3, 4, 5
    h, w, g = rng.standard_normal((T, M)), rng.standard_normal((V, M)), rng.standard_normal((T, V))
    lg = lm_head_forward(h, w)
    for t in range(T):
        for v in range(V):
            assert np.isclose(lg[t, v], sum(h[t, m] * w[v, m] for m in range(M)))
    dh, dw = lm_head_backward(h, w, g)
    # <lm_head(h), g> = <h, dh> = <w, dw> (both adjoints)
    assert np.isclose(np.sum(lg * g), np.sum(h * dh)) and np.isclose(np.sum(lg * g), np.sum(w * dw))
