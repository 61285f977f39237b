"""Pins tests/torch_ref.py — the numerics reference of the bf16 parity tests
(test_gpu_bf16_shapes.py) — to the reference's golden vectors: run in fp32 and
fp64 on init_model weights (taken from the oracle, itself bit-exact against
init_model) in the reference configuration (MHA, tied head, rope base 10000),
it must reproduce the unmodified reference's logits and hidden states
(oracle/_ref/ref_dump: proj/tests/test_model.cpp:61-68 KAT, prefill, fuzzy
forwards at lp 1-4). CPU only."""
import json
import os
from types import SimpleNamespace

import numpy as np
import pytest
import torch

from oracle import oracle as O
from tests import torch_ref

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
NUM = json.load(open(os.path.join(GOLDEN, "ref_numerics.json")))
TOL = 2e-4  # relative to max |logit| (fp32 reference, different summation order)


def _weights(cfgj, dtype):
    m = O.Model(O.ModelConfig(**cfgj))
    W = {"embedding": m.tensor("embedding"), "final_norm_gain": m.tensor("final_norm_gain")[0]}
    for l in range(cfgj["n_layers"]):
        for n in ("wq", "wk", "wv", "wo", "w_gate", "w_up", "w_down"):
            W[f"{n}.{l}"] = m.tensor(n, l)
        for n in ("attn_norm_gain", "mlp_norm_gain"):
            W[f"{n}.{l}"] = m.tensor(n, l)[0]
    cfg = SimpleNamespace(**cfgj, n_kv_heads=cfgj["n_heads"], rope_theta=10000.0, tied_head=True)
    return {k: torch.from_numpy(np.ascontiguousarray(v)).to(dtype) for k, v in W.items()}, cfg


def _toks(prompt):
    return [256] + list(prompt.encode())


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_golden_argmax_110(dtype):
    g = NUM["golden_argmax"]
    W, cfg = _weights(g["config"], dtype)
    logits, _ = torch_ref.forward(W, cfg, _toks(g["prompt"]))
    last = logits[-1].double().numpy()
    assert int(last.argmax()) == g["argmax"] == 110
    want = np.asarray(g["logits"])
    assert np.abs(last - want).max() <= TOL * np.abs(want).max()


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_prefill_logits_and_hidden(dtype):
    g = NUM["prefill_kv"]
    W, cfg = _weights(g["config"], dtype)
    toks = _toks(g["prompt"])
    logits, hidden = torch_ref.forward(W, cfg, toks)
    want_l = np.asarray(g["logits"]).reshape(len(toks), -1)
    want_h = np.asarray(g["hidden"]).reshape(len(toks), -1)
    assert np.abs(logits.double().numpy() - want_l).max() <= TOL * np.abs(want_l).max()
    assert np.abs(hidden.double().numpy() - want_h).max() <= TOL * np.abs(want_h).max()


@pytest.mark.parametrize("lp", [1, 2, 3, 4])
def test_fuzzy_forward(lp):
    g = NUM["fuzzy"]
    W, cfg = _weights(g["config"], torch.float64)
    plan = [[int(x) for x in range(int(s.split("-")[0]), int(s.split("-")[-1]) + 1)]
            for s in g[f"lp{lp}"]["plan"].split("|")]
    logits, hidden = torch_ref.forward(W, cfg, g["tokens"], plan)
    want_l = np.asarray(g[f"lp{lp}"]["logits"]).reshape(len(g["tokens"]), -1)
    want_h = np.asarray(g[f"lp{lp}"]["hidden"]).reshape(len(g["tokens"]), -1)
    assert np.abs(logits.numpy() - want_l).max() <= TOL * np.abs(want_l).max()
    assert np.abs(hidden.numpy() - want_h).max() <= TOL * np.abs(want_h).max()


def test_tree_rows_mask_matches_reference_kat():
    """tree_rows against the tree_commit fixture's shape rules: a staged
    child sees the committed prefix and its ancestors only."""
    pos, mask = torch_ref.tree_rows(3, [-1, 0, 0, 1])
    assert pos.tolist() == [0, 1, 2, 3, 4, 4, 5]
    assert mask[6].tolist() == [True, True, True, True, True, False, True]
    assert mask[5].tolist() == [True, True, True, True, False, True, False]
