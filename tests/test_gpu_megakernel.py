"""Decode megakernel (csrc/decode_mk.cu) parity.

A decode pass of T <= 8 rows on one GPU runs as ONE persistent launch that
executes the same GEMV units (same stream-K plan, warp and k-chunk reduction
order, fused epilogues) and the same attention items as the per-kernel path.
Bar: BITWISE equality of logits, hidden rows, K/V cache rows and emitted
tokens with the megakernel on (default) and off (ESPEC_MK=0), so every bf16
tolerance and losslessness result of test_gpu_parity.py carries over.
"""
import os
from dataclasses import replace

import numpy as np
import pytest

from paper_2502_02493_b200 import espec as E

pytestmark = pytest.mark.gpu


def _pair(d_model=512, n_layers=6, keep=4, n_heads=8, n_kv=2, dh=64, f=1536, vocab=4096, seed=5, max_pos=1024):
    base = E.ModelConfig(vocab_size=vocab, d_model=d_model, n_layers=n_layers, n_heads=n_heads, n_kv_heads=n_kv,
                         d_head=dh, d_mlp=f, max_positions=max_pos, seed=seed, rope_theta=500000.0,
                         tied_head=False, weight_dtype=E.BF16, kv_dtype=E.BF16)
    return base, replace(base, n_layers=keep, seed=seed + 100)


PAIRS = {
    "dh64": _pair(),
    # Llama-3 head shape: GQA group 8, d_head 128
    "dh128_g8": _pair(d_model=1024, n_layers=4, keep=4, n_heads=16, n_kv=2, dh=128, f=2816, vocab=8192, seed=9),
}


def _engine(base, draft, run, mk):
    # the megakernel runs every GEMV on the (K, N)-only plan; compare against
    # the per-kernel path with the drafter on that plan too (ESPEC_WIDE_DRAFT=0)
    os.environ["ESPEC_MK"] = "1" if mk else "0"
    os.environ["ESPEC_WIDE_DRAFT"] = "0"
    try:
        eng = E.Engine(base, draft, run)
    finally:
        os.environ.pop("ESPEC_MK", None)
        os.environ.pop("ESPEC_WIDE_DRAFT", None)
    eng.init_weights(E.Engine.BASE, base.seed, parity=False)
    eng.init_weights(E.Engine.DRAFT, draft.seed, parity=False)
    return eng


@pytest.mark.parametrize("pair", sorted(PAIRS))
@pytest.mark.parametrize("T", [1, 3, 6, 8])
def test_forward_bitwise_equal_with_and_without_megakernel(pair, T):
    base, draft = PAIRS[pair]
    rng = np.random.default_rng(T)
    toks = [int(t) for t in rng.integers(0, base.vocab_size, size=T)]
    res = {}
    for mk in (True, False):
        eng = _engine(base, draft, E.RunConfig(n=5, lp_size=2), mk)
        out = []
        for which, plan in ((E.Engine.BASE, None), (E.Engine.DRAFT, None), (E.Engine.DRAFT, "lp=2"),
                            (E.Engine.DRAFT, "lp=3")):
            logits, hidden = eng.forward(which, toks, plan=plan)
            k, v, n = eng.cache_view(which, 1, 0, T)
            out.append((logits, hidden, k, v))
        res[mk] = out
        eng.close()
    for a, b in zip(res[True], res[False]):
        for x, y in zip(a, b):
            assert np.array_equal(x, y)


@pytest.mark.parametrize("pair", sorted(PAIRS))
def test_generate_tokens_equal_with_and_without_megakernel(pair):
    """Greedy EasySpec over a 300-token prompt (tcgen05 prefill, then decode
    passes whose context spans several 64-row pages and split-KV chunks)."""
    base, draft = PAIRS[pair]
    rng = np.random.default_rng(11)
    prompt = [int(t) for t in rng.integers(0, base.vocab_size, size=300)]
    outs = {}
    for alg in ("vanilla", "easyspec"):
        for mk in (True, False):
            eng = _engine(base, draft, E.RunConfig(algorithm=alg, n=5, lp_size=2, max_new_tokens=40), mk)
            outs[(alg, mk)], _ = eng.generate_tokens(prompt)
            eng.close()
    assert outs[("easyspec", True)] == outs[("easyspec", False)]
    assert outs[("vanilla", True)] == outs[("vanilla", False)]
    assert outs[("vanilla", True)] == outs[("easyspec", True)]  # losslessness through the megakernel


def test_sampled_tree_tokens_equal_with_and_without_megakernel():
    """T = 0.8 rejection sampling over a [2,2,1] tree: draft levels (T = 2, 4
    rows) run in the megakernel, the 13-row verify on the per-kernel path."""
    base, draft = PAIRS["dh64"]
    outs = {}
    for mk in (True, False):
        run = E.RunConfig(algorithm="easyspec", n=3, widths=[2, 2, 1], lp_size=2, temperature=0.8,
                          max_new_tokens=32, seed=7)
        eng = _engine(base, draft, run, mk)
        outs[mk], _ = eng.generate(b"sampled tree through the megakernel")
        eng.close()
    assert outs[True] == outs[False]


def test_megakernel_is_one_launch_per_pass():
    base, draft = PAIRS["dh64"]
    launches = {}
    for mk in (True, False):
        eng = _engine(base, draft, E.RunConfig(algorithm="easyspec", n=5, lp_size=2, max_new_tokens=64), mk)
        eng.begin(list(range(1, 20)))
        eng.step()
        eng.reset_kernel_launches()
        for _ in range(3):
            eng.step()
        launches[mk] = eng.kernel_launches()
        eng.close()
    # per iteration: calibrate + 4 fuzzy draft passes + 1 verify pass = 6
    # megakernels, 6 heads, the embed of nothing else and one accept kernel
    assert launches[True] <= 3 * 16, launches
    assert launches[True] * 4 < launches[False], launches
