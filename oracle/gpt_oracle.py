"""TEST INFRASTRUCTURE ONLY -- numpy fp64 restatement of Chimera training of a
GPT-2-style transformer under the reference oracle's Engine semantics.

The reference (proj/src/oracle.cpp) has no transformer; this file restates its
Engine (oracle.cpp:162-300) for a real stage model and is the numerical checker of
the sm_100a GPT stage executor:
  * replay order = unit-tick list schedule sorted by (start, worker, index)
    (oracle.cpp:312-327), computed with the C restatement toy_oracle.c
    (toy_list_schedule, listsched.hpp:52-163);
  * per task, a loop over data-parallel replicas r (oracle.cpp:337,340);
  * stash keyed by (r, pipeline, micro, stage) (oracle.cpp:174,236-237);
  * sample map (r*N + m)*B (oracle.cpp:200); loss = mean over all B_hat*seq tokens
    (so the per-sample gradient scale is 1/B_hat as in oracle.cpp:330);
  * gradients per (r, pipeline) copy, summed over all 2f*W copies, then plain SGD
    on every copy (apply_stage_update, oracle.cpp:283-299).
Model: pre-LN GPT-2 block (LN eps 1e-5, tanh-GELU, causal softmax attention with
head dim 64, untied LM head over a padded vocabulary, mean softmax cross-entropy);
same per-stage flat parameter layout as the product (checked by the tests).
"Parity pinning": the reference cannot run this model, so the oracle is pinned by
the reference's own property (pipelined == sequential SGD, <= 1e-10 in fp64) and by
central finite differences (tests/test_gpt_oracle.py).
"""
from __future__ import annotations

import json
import math
from dataclasses import dataclass

import numpy as np


@dataclass
class Shape:
    n_layer: int = 8
    hidden: int = 256
    heads: int = 4
    ffn: int = 1024
    seq: int = 128
    vocab: int = 1024
    vocab_padded: int = 1024
    causal: bool = True
    stage_layers: tuple = ()


def stage_layout(m: Shape, D: int, s: int):
    """[(name, offset, rows, cols, init)] + total, 64-element aligned (product convention)."""
    out, total = [], 0
    h, f = m.hidden, m.ffn

    def add(name, rows, cols, init):
        nonlocal total
        out.append((name, total, rows, cols, init))
        total += (rows * cols + 63) // 64 * 64

    parts = list(m.stage_layers) or [m.n_layer // D] * D
    per, first = parts[s], sum(parts[:s])
    if s == 0:
        add("wte", m.vocab_padded, h, "normal")
        add("wpe", m.seq, h, "normal")
    for l in range(per):
        p = f"h{first + l}."
        add(p + "ln1.g", 1, h, "one"); add(p + "ln1.b", 1, h, "zero")
        add(p + "attn.w_qkv", 3 * h, h, "normal"); add(p + "attn.b_qkv", 1, 3 * h, "zero")
        add(p + "attn.w_o", h, h, "normal"); add(p + "attn.b_o", 1, h, "zero")
        add(p + "ln2.g", 1, h, "one"); add(p + "ln2.b", 1, h, "zero")
        add(p + "mlp.w_fc1", f, h, "normal"); add(p + "mlp.b_fc1", 1, f, "zero")
        add(p + "mlp.w_fc2", h, f, "normal"); add(p + "mlp.b_fc2", 1, h, "zero")
    if s == D - 1:
        add("lnf.g", 1, h, "one"); add("lnf.b", 1, h, "zero")
        add("lm_head", m.vocab_padded, h, "normal")
    return out, total


def unpack(flat, layout):
    return {n: flat[o:o + r * c].reshape(r, c) if r > 1 else flat[o:o + c] for n, o, r, c, _ in layout}


def pack(d, layout, total):
    flat = np.zeros(total)
    for n, o, r, c, _ in layout:
        flat[o:o + r * c] = np.asarray(d[n]).reshape(-1)
    return flat


# ----------------------------------------------------------------- layer math --
C0, C1 = math.sqrt(2.0 / math.pi), 0.044715


def gelu(u):
    return 0.5 * u * (1.0 + np.tanh(C0 * (u + C1 * u ** 3)))


def gelu_grad(u):
    t = np.tanh(C0 * (u + C1 * u ** 3))
    return 0.5 * (1 + t) + 0.5 * u * (1 - t * t) * C0 * (1 + 3 * C1 * u * u)


def ln_fwd(x, g, b):
    mu = x.mean(-1, keepdims=True)
    var = ((x - mu) ** 2).mean(-1, keepdims=True)
    rs = 1.0 / np.sqrt(var + 1e-5)
    xh = (x - mu) * rs
    return xh * g + b, (xh, rs)


def ln_bwd(dy, cache, g):
    xh, rs = cache
    gg = dy * g
    dx = rs * (gg - gg.mean(-1, keepdims=True) - xh * (gg * xh).mean(-1, keepdims=True))
    return dx, (dy * xh).sum(0), dy.sum(0)


def attn_fwd(qkv, B, s, H, causal):
    d = 64
    q, k, v = qkv.reshape(B, s, 3, H, d).transpose(2, 0, 3, 1, 4)  # [B,H,s,d]
    sc = q @ k.transpose(0, 1, 3, 2) / 8.0
    if causal:
        sc = np.where(np.triu(np.ones((s, s), bool), 1), -np.inf, sc)
    sc = sc - sc.max(-1, keepdims=True)
    p = np.exp(sc)
    p /= p.sum(-1, keepdims=True)
    o = p @ v
    return o.transpose(0, 2, 1, 3).reshape(B * s, H * d), (q, k, v, p)


def attn_bwd(do, cache, B, s, H):
    q, k, v, p = cache
    d = 64
    do = do.reshape(B, s, H, d).transpose(0, 2, 1, 3)
    dv = p.transpose(0, 1, 3, 2) @ do
    dp = do @ v.transpose(0, 1, 3, 2)
    ds = p * (dp - (dp * p).sum(-1, keepdims=True)) / 8.0
    dq = ds @ k
    dk = ds.transpose(0, 1, 3, 2) @ q
    return np.stack([dq, dk, dv], 0).transpose(1, 3, 0, 2, 4).reshape(B * s, 3 * H * d)


class StageModel:
    """Forward/backward of one pipeline stage on one micro-batch (fp64)."""

    def __init__(self, m: Shape, D: int, s: int):
        self.m, self.D, self.s = m, D, s
        self.layout, self.total = stage_layout(m, D, s)
        parts = list(m.stage_layers) or [m.n_layer // D] * D
        self.per, self.first = parts[s], sum(parts[:s])

    def forward(self, P, x_or_tok, labels, B, loss_scale):
        m = self.m
        h, H, seq = m.hidden, m.heads, m.seq
        cache = {}
        if self.s == 0:
            tok = x_or_tok
            x = P["wte"][tok] + P["wpe"][np.arange(len(tok)) % seq]
            cache["tok"] = tok
        else:
            x = x_or_tok
        for l in range(self.per):
            p = f"h{self.first + l}."
            h1, c1 = ln_fwd(x, P[p + "ln1.g"], P[p + "ln1.b"])
            qkv = h1 @ P[p + "attn.w_qkv"].T + P[p + "attn.b_qkv"]
            a, ca = attn_fwd(qkv, B, seq, H, m.causal)
            x2 = a @ P[p + "attn.w_o"].T + P[p + "attn.b_o"] + x
            h2, c2 = ln_fwd(x2, P[p + "ln2.g"], P[p + "ln2.b"])
            u = h2 @ P[p + "mlp.w_fc1"].T + P[p + "mlp.b_fc1"]
            g = gelu(u)
            y = g @ P[p + "mlp.w_fc2"].T + P[p + "mlp.b_fc2"] + x2
            cache[l] = (x, h1, c1, a, ca, x2, h2, c2, u, g)
            x = y
        loss = None
        if self.s == self.D - 1:
            hf, cf = ln_fwd(x, P["lnf.g"], P["lnf.b"])
            logits = hf @ P["lm_head"].T
            lg = logits[:, :m.vocab]
            mx = lg.max(-1, keepdims=True)
            lse = mx[:, 0] + np.log(np.exp(lg - mx).sum(-1))
            loss = float((lse - lg[np.arange(len(labels)), labels]).sum() * loss_scale)
            dl = np.exp(lg - lse[:, None])
            dl[np.arange(len(labels)), labels] -= 1.0
            dlog = np.zeros_like(logits)
            dlog[:, :m.vocab] = dl * loss_scale
            cache["head"] = (x, hf, cf, dlog)
        return x, loss, cache

    def backward(self, P, G, cache, dy, B):
        m = self.m
        H, seq = m.heads, m.seq
        if self.s == self.D - 1:
            x, hf, cf, dlog = cache["head"]
            G["lm_head"] += dlog.T @ hf
            dhf = dlog @ P["lm_head"]
            dy, dg, db = ln_bwd(dhf, cf, P["lnf.g"])
            G["lnf.g"] += dg
            G["lnf.b"] += db
        for l in reversed(range(self.per)):
            p = f"h{self.first + l}."
            x, h1, c1, a, ca, x2, h2, c2, u, g = cache[l]
            G[p + "mlp.b_fc2"] += dy.sum(0)
            G[p + "mlp.w_fc2"] += dy.T @ g
            du = (dy @ P[p + "mlp.w_fc2"]) * gelu_grad(u)
            G[p + "mlp.b_fc1"] += du.sum(0)
            G[p + "mlp.w_fc1"] += du.T @ h2
            dh2 = du @ P[p + "mlp.w_fc1"]
            d, dg, db = ln_bwd(dh2, c2, P[p + "ln2.g"])
            dx2 = dy + d
            G[p + "ln2.g"] += dg
            G[p + "ln2.b"] += db
            G[p + "attn.b_o"] += dx2.sum(0)
            G[p + "attn.w_o"] += dx2.T @ a
            da = dx2 @ P[p + "attn.w_o"]
            dqkv = attn_bwd(da, ca, B, seq, H)
            G[p + "attn.b_qkv"] += dqkv.sum(0)
            G[p + "attn.w_qkv"] += dqkv.T @ h1
            dh1 = dqkv @ P[p + "attn.w_qkv"]
            d, dg, db = ln_bwd(dh1, c1, P[p + "ln1.g"])
            dy = dx2 + d
            G[p + "ln1.g"] += dg
            G[p + "ln1.b"] += db
        if self.s == 0:
            tok = cache["tok"]
            np.add.at(G["wte"], tok, dy)
            G["wpe"] += dy.reshape(B, seq, -1).sum(0)
            return None
        return dy


def replay_order(schedule: dict):
    """Unit-tick list schedule via the C restatement (toy_oracle.c), sorted by
    (start, worker, index) -- oracle.cpp:312-327."""
    from .libs import ToyLib
    cfg = schedule["config"]
    halved = cfg["scheme"] == "chimera" and cfg["scaling"] == "backward-halving" and cfg["N"] > cfg["D"]
    st, _, _ = ToyLib().list_schedule(schedule, 2.0 if halved else 1.0, 2.0)
    items, k = [], 0
    for w, wl in enumerate(schedule["per_worker"]):
        for i in range(len(wl)):
            items.append((st[k], w, i))
            k += 1
    items.sort()
    return [(w, i) for _, w, i in items]


def run_iteration(schedule: dict, m: Shape, params, tokens, labels, lr):
    """One pipelined iteration.  params: list of flat fp64 vectors per stage.
    Returns (new params, mean loss, summed gradient per stage, peak stash per worker)."""
    cfg = schedule["config"]
    D, W, N, B = cfg["D"], cfg["W"], cfg["N"], cfg["B"]
    P = 1 + max(t["pipeline_id"] for wl in schedule["per_worker"] for t in wl)
    models = [StageModel(m, D, s) for s in range(D)]
    Pv = [unpack(params[s], models[s].layout) for s in range(D)]
    grads = {(r, p, s): {n: np.zeros((rr, cc)) if rr > 1 else np.zeros(cc)
                         for n, _, rr, cc, _ in models[s].layout}
             for r in range(W) for p in range(P) for s in range(D)}
    stash, outs, gin = {}, {}, {}
    live = [0] * D
    peak = [0] * D
    seq = m.seq
    scale = 1.0 / (W * N * B * seq)
    loss = 0.0
    for w, i in replay_order(schedule):
        t = schedule["per_worker"][w][i]
        if t["kind"] not in ("Forward", "Backward"):
            continue
        p, mb, s = t["pipeline_id"], t["micro_batch"], t["stage"]
        for r in range(W):
            rows = slice((r * N + mb) * B * seq, (r * N + mb + 1) * B * seq)
            if t["kind"] == "Forward":
                inp = tokens[rows] if s == 0 else outs[(r, p, mb, s - 1)]
                y, ls, cache = models[s].forward(Pv[s], inp, labels[rows], B, scale)
                stash[(r, p, mb, s)] = cache
                outs[(r, p, mb, s)] = y
                if ls is not None:
                    loss += ls
                if r == 0:
                    live[w] += 1
                    peak[w] = max(peak[w], live[w])
            else:
                cache = stash.pop((r, p, mb, s))
                dy = None if s == D - 1 else gin.pop((r, p, mb, s))
                dx = models[s].backward(Pv[s], grads[(r, p, s)], cache, dy, B)
                if s > 0:
                    gin[(r, p, mb, s - 1)] = dx
                if r == 0:
                    live[w] -= 1
    new, gsum = [], []
    for s in range(D):
        tot = {n: sum(grads[(r, p, s)][n] for r in range(W) for p in range(P)) for n in Pv[s]}
        gsum.append(pack(tot, models[s].layout, models[s].total))
        new.append(params[s] - lr * gsum[-1])
    return new, loss, gsum, peak


def sequential_sgd(m: Shape, D: int, params, tokens, labels, lr, B_hat):
    """Plain mini-batch SGD over the whole batch (oracle.cpp:125-151 analogue)."""
    models = [StageModel(m, D, s) for s in range(D)]
    Pv = [unpack(params[s], models[s].layout) for s in range(D)]
    G = [{n: np.zeros((rr, cc)) if rr > 1 else np.zeros(cc) for n, _, rr, cc, _ in mm.layout} for mm in models]
    scale = 1.0 / (B_hat * m.seq)
    x, loss, caches = tokens, 0.0, []
    for s in range(D):
        x, ls, c = models[s].forward(Pv[s], x, labels, B_hat, scale)
        caches.append(c)
        if ls is not None:
            loss += ls
    dy = None
    for s in reversed(range(D)):
        dy = models[s].backward(Pv[s], G[s], caches[s], dy, B_hat)
    gsum = [pack(G[s], models[s].layout, models[s].total) for s in range(D)]
    return [params[s] - lr * gsum[s] for s in range(D)], loss, gsum


def init_params(m: Shape, D: int, seed: int = 0):
    """N(0, 0.02) matrices, zero biases, unit LN gains, fp64."""
    out = []
    for s in range(D):
        layout, total = stage_layout(m, D, s)
        rng = np.random.default_rng([seed, s])
        flat = np.zeros(total)
        for n, o, r, c, init in layout:
            if init == "normal":
                flat[o:o + r * c] = rng.standard_normal(r * c) * 0.02
            elif init == "one":
                flat[o:o + r * c] = 1.0
        out.append(flat)
    return out


def synthetic_tokens(m: Shape, n_samples: int, seed: int = 0):
    rng = np.random.default_rng(seed)
    seqs = rng.integers(0, m.vocab, size=(n_samples, m.seq + 1), dtype=np.int64)
    return seqs[:, :-1].reshape(-1).astype(np.int32), seqs[:, 1:].reshape(-1).astype(np.int32)


def schedule_dict(text: str) -> dict:
    return json.loads(text)
