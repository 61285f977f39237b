"""Plain PyTorch restatement of the model forward, the numerics reference for
the bf16 kernels. Test infrastructure only.

Follows proj/src/model.cpp:114-215 (attention_forward / mlp_forward /
lm_logits), proj/src/matrix.cpp:118-137 (rms_norm) and 159-194 (apply_rope:
pairs (2i, 2i+1), angle pos * theta^(-2i/dh) in double), extended with GQA,
an untied head and a rope base, and evaluated in any dtype (fp64 for the
bf16 parity tests). `forward_rows` takes explicit positions and a visibility
mask, i.e. the tree passes of verify_stage / draft_tree
(proj/src/orchestrator.cpp:333-388, proj/src/kv_cache.cpp:43-60).
tests/test_torch_ref.py pins it to the reference's golden vectors.
"""
import math

import torch


def rope(x, pos, dh, theta):
    # x: [T, H*dh]; rotation in fp64, result in x's dtype
    T = x.shape[0]
    xv = x.view(T, -1, dh // 2, 2)
    inv = torch.tensor([theta ** (-2.0 * p / dh) for p in range(dh // 2)], dtype=torch.float64, device=x.device)
    ang = pos.to(torch.float64)[:, None] * inv[None, :]
    c = torch.cos(ang)[:, None, :]
    s = torch.sin(ang)[:, None, :]
    if x.dtype != torch.float64:
        c, s = c.float().to(x.dtype), s.float().to(x.dtype)
    x0, x1 = xv[..., 0], xv[..., 1]
    return torch.stack([x0 * c - x1 * s, x0 * s + x1 * c], -1).view(T, -1)


def rmsnorm(h, g, eps):
    return h / torch.sqrt((h * h).mean(-1, keepdim=True) + eps) * g


def _rb(x, on):
    """bf16 round trip (the engine's storage / tensor-core operand points)."""
    return x.to(torch.bfloat16).to(x.dtype) if on else x


def _attn(W, cfg, l, hn, pos, mask, past=None, kv_out=None, rb=False):
    T = hn.shape[0]
    H, Hkv, dh = cfg.n_heads, cfg.n_kv_heads or cfg.n_heads, cfg.d_head
    G = H // Hkv
    hn = _rb(hn, rb)
    q = _rb(rope(hn @ W[f"wq.{l}"], pos, dh, cfg.rope_theta), rb).view(T, H, dh)
    k = _rb(rope(hn @ W[f"wk.{l}"], pos, dh, cfg.rope_theta), rb).view(T, Hkv, dh)
    v = _rb(hn @ W[f"wv.{l}"], rb).view(T, Hkv, dh)
    if kv_out is not None:
        kv_out[l] = (k, v)
    if past is not None:  # cached rows of earlier passes (the KV cache)
        k = torch.cat([past[l][0], k], 0)
        v = torch.cat([past[l][1], v], 0)
    k = k.repeat_interleave(G, dim=1)
    v = v.repeat_interleave(G, dim=1)
    sc = torch.einsum("thd,shd->hts", q, k) / math.sqrt(dh)
    sc = sc.masked_fill(~mask[None], float("-inf"))
    if rb:  # unnormalised probabilities enter the PV product in bf16, the sum in full precision
        e = torch.exp(sc - sc.amax(-1, keepdim=True))
        p = _rb(e, True) / e.sum(-1, keepdim=True)
    else:
        p = torch.softmax(sc, -1)
    o = torch.einsum("hts,shd->thd", p, v).reshape(T, H * dh)
    return _rb(o, rb) @ W[f"wo.{l}"]


def forward_rows(W, cfg, tokens, pos, mask, plan=None, head_rows=None, past=None, kv_out=None, bf16_acts=False):
    """One pass over rows: tokens [T], rotary positions [T], mask [T, P + T]
    (row i may attend to cached row j < P or pass row j - P). plan: list of
    layer groups (forward_fuzzy: every attention layer of a group reads the
    group's entry state, proj/src/draft_engine.cpp:64-133). past: per-layer
    (k, v) of P cached rows; kv_out (dict) receives this pass's (k, v).
    bf16_acts: round to bf16 where the engine stores or feeds tensor cores
    (GEMV inputs, q / K / V, attention probabilities and output, SiLU output).
    Returns (logits of head_rows, hidden)."""
    dev = W["embedding"].device
    tok = torch.as_tensor(tokens, device=dev)
    pos = torch.as_tensor(pos, device=dev)
    mask = torch.as_tensor(mask, device=dev)
    h = W["embedding"][tok]
    groups = plan or [[l] for l in range(cfg.n_layers)]
    for g in groups:
        entry = h
        outs = [_attn(W, cfg, l, rmsnorm(entry, W[f"attn_norm_gain.{l}"], cfg.norm_eps), pos, mask, past, kv_out,
                      bf16_acts) for l in g]
        for l, a in zip(g, outs):
            h = h + a
            mn = _rb(rmsnorm(h, W[f"mlp_norm_gain.{l}"], cfg.norm_eps), bf16_acts)
            gt = mn @ W[f"w_gate.{l}"]
            up = mn @ W[f"w_up.{l}"]
            h = h + _rb(gt / (1 + torch.exp(-gt)) * up, bf16_acts) @ W[f"w_down.{l}"]
    hr = h if head_rows is None else h[head_rows]
    hn = _rb(rmsnorm(hr, W["final_norm_gain"], cfg.norm_eps), bf16_acts)
    head = W["embedding"].t() if cfg.tied_head else W["head"]
    return hn @ head, h


def forward(W, cfg, tokens, plan=None):
    """Chain prefill of `tokens` from an empty cache; returns (logits, hidden)."""
    T = len(tokens)
    dev = W["embedding"].device
    mask = torch.tril(torch.ones(T, T, dtype=torch.bool, device=dev))
    return forward_rows(W, cfg, tokens, torch.arange(T, device=dev), mask, plan)


def tree_rows(n_prompt, parents):
    """Positions and mask of a prompt (causal chain) followed by tree rows:
    parents[j] = -1 (child of the prompt tail) or an earlier tree row. A tree
    row sees the whole prompt and its ancestors (itself included); its
    position is n_prompt + depth - 1 (KvCache::position_of,
    proj/src/kv_cache.cpp:167-171)."""
    T = len(parents)
    N = n_prompt + T
    mask = torch.zeros(N, N, dtype=torch.bool)
    mask[:n_prompt, :n_prompt] = torch.tril(torch.ones(n_prompt, n_prompt, dtype=torch.bool))
    pos = list(range(n_prompt))
    depth = []
    for j, p in enumerate(parents):
        depth.append(1 if p < 0 else depth[p] + 1)
        pos.append(n_prompt + depth[j] - 1)
        r = n_prompt + j
        mask[r, :n_prompt] = True
        a = j
        while a >= 0:
            mask[r, n_prompt + a] = True
            a = parents[a]
    return torch.tensor(pos), mask
