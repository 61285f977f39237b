"""Plain PyTorch fp32 restatement of the model forward for numerics tests of
the bf16 kernels (GQA, rotary pairs (2i, 2i+1) as in proj/src/matrix.cpp:159-194).
Test infrastructure only."""
import math

import torch


def rope(x, pos, dh, theta):
    # x: [T, H*dh]
    T = x.shape[0]
    xv = x.view(T, -1, dh // 2, 2)
    inv = torch.tensor([theta ** (-2.0 * p / dh) for p in range(dh // 2)], dtype=torch.float64)
    ang = pos.double()[:, None] * inv[None, :]
    c, s = torch.cos(ang).float()[:, None, :], torch.sin(ang).float()[:, None, :]
    x0, x1 = xv[..., 0], xv[..., 1]
    return torch.stack([x0 * c - x1 * s, x0 * s + x1 * c], -1).view(T, -1)


def rmsnorm(h, g, eps):
    return h / torch.sqrt((h * h).mean(-1, keepdim=True) + eps) * g


def forward(W, cfg, tokens, plan=None):
    """W: dict of fp32 tensors in the reference layout. Chain prefill of
    `tokens` from an empty cache; returns (logits, hidden)."""
    d, H, Hkv, dh = cfg.d_model, cfg.n_heads, cfg.n_kv_heads or cfg.n_heads, cfg.d_head
    G = H // Hkv
    T = len(tokens)
    pos = torch.arange(T)
    h = W["embedding"][torch.tensor(tokens)]
    groups = plan or [[l] for l in range(cfg.n_layers)]
    mask = torch.tril(torch.ones(T, T, dtype=torch.bool))
    for g in groups:
        entry = h
        outs = []
        for l in g:
            hn = rmsnorm(entry, W[f"attn_norm_gain.{l}"], cfg.norm_eps)
            q = rope(hn @ W[f"wq.{l}"], pos, dh, cfg.rope_theta).view(T, H, dh)
            k = rope(hn @ W[f"wk.{l}"], pos, dh, cfg.rope_theta).view(T, Hkv, dh)
            v = (hn @ W[f"wv.{l}"]).view(T, Hkv, dh)
            k = k.repeat_interleave(G, dim=1)
            v = v.repeat_interleave(G, dim=1)
            sc = torch.einsum("thd,shd->hts", q, k) / math.sqrt(dh)
            sc = sc.masked_fill(~mask[None], float("-inf"))
            p = torch.softmax(sc, -1)
            o = torch.einsum("hts,shd->thd", p, v).reshape(T, H * dh)
            outs.append(o @ W[f"wo.{l}"])
        for l, a in zip(g, outs):
            h = h + a
            mn = rmsnorm(h, W[f"mlp_norm_gain.{l}"], cfg.norm_eps)
            gt = mn @ W[f"w_gate.{l}"]
            up = mn @ W[f"w_up.{l}"]
            h = h + (gt / (1 + torch.exp(-gt)) * up) @ W[f"w_down.{l}"]
    hn = rmsnorm(h, W["final_norm_gain"], cfg.norm_eps)
    head = W["embedding"].t() if cfg.tied_head else W["head"]
    return hn @ head, h
