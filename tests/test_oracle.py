"""Pins the CPU oracle (oracle/espec_oracle.c) to the reference.

Every comparison here is bit-exact: the fixtures in tests/golden/ were written
by the unmodified reference core (oracle/_ref/ref_dump), and the oracle
restates the same fp32 operation order. CPU only.
"""
import json
import os

import numpy as np
import pytest

from oracle import oracle as O

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _load(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


NUM = _load("ref_numerics.json")
GEN = _load("ref_generate.json")


def _cfg(j):
    return O.ModelConfig(**{k: j[k] for k in ("vocab_size", "d_model", "n_layers", "n_heads", "d_head",
                                               "d_mlp", "max_positions", "norm_eps", "seed")})


def _models(case):
    base = O.Model(_cfg(case["base"]))
    if case["draft_seed"]:
        dc = _cfg(case["base"])
        dc.n_layers, dc.seed = case["keep"], case["draft_seed"]
        return base, O.Model(dc)
    return base, (base if case["keep"] == 0 else base.truncated(case["keep"]))


def _run(case):
    r = case["run"]
    return O.RunConfig(algorithm=r["algorithm"], n=r["n"], widths=r["widths"], lp_size=r["lp_size"],
                       plan_override=r["plan_override"] or None, temperature=r["temperature"],
                       max_new_tokens=r["max_new_tokens"], seed=r["seed"], calibration=r["calibration"])


def test_init_model_matches_reference_stream():
    for probe in NUM["init"]:
        m = O.Model(_cfg(probe["config"]))
        emb = m.tensor("embedding")
        assert emb.astype(np.float64).sum() == probe["embedding_sum"]
        assert np.array_equal(emb.ravel()[:8], np.asarray(probe["embedding_head"], np.float32))
        for layer, want in enumerate(probe["layers"]):
            for name in ("wq", "wk", "wv", "wo", "w_gate", "w_up", "w_down"):
                assert m.tensor(name, layer).astype(np.float64).sum() == want[name], (layer, name)


def test_golden_argmax_110():
    """proj/tests/test_model.cpp:61-68."""
    g = NUM["golden_argmax"]
    m = O.Model(_cfg(g["config"]))
    _, logits, _, _ = m.prefill(O.tokenize(b"golden"))
    assert int(np.argmax(logits[-1])) == 110 == g["argmax"]
    assert np.array_equal(logits[-1], np.asarray(g["logits"], np.float32))


def test_prefill_kv_hidden_logits_bit_exact():
    g = NUM["prefill_kv"]
    m = O.Model(_cfg(g["config"]))
    h, logits, k, v = m.prefill(O.tokenize(g["prompt"].encode()))
    assert np.array_equal(h.ravel(), np.asarray(g["hidden"], np.float32))
    assert np.array_equal(logits.ravel(), np.asarray(g["logits"], np.float32))
    for layer in range(2):
        assert np.array_equal(k[layer].ravel(), np.asarray(g["kv"][layer]["k"], np.float32))
        assert np.array_equal(v[layer].ravel(), np.asarray(g["kv"][layer]["v"], np.float32))


@pytest.mark.parametrize("lp", [1, 2, 3, 4])
def test_fuzzy_forward_bit_exact(lp):
    g = NUM["fuzzy"]
    m = O.Model(_cfg(g["config"]))
    h, logits, _, _ = m.prefill(g["tokens"], plan=f"lp={lp}")
    assert O.plan_groups(8, lp) == g[f"lp{lp}"]["plan"]
    assert np.array_equal(h.ravel(), np.asarray(g[f"lp{lp}"]["hidden"], np.float32))
    assert np.array_equal(logits.ravel(), np.asarray(g[f"lp{lp}"]["logits"], np.float32))


def test_all_singleton_fuzzy_equals_sequential():
    """Criterion 3 (proj/tests/acceptance_main.cpp:186-217)."""
    m = O.Model(O.tiny_config(6, 63))
    rng = np.random.default_rng(64)
    for _ in range(10):
        toks = list(rng.integers(0, 256, size=int(rng.integers(1, 6))))
        a = m.prefill(toks, plan="lp=1")[0]
        b = m.prefill(toks)[0]
        assert np.array_equal(a, b)


def test_layer_plans():
    for p in NUM["plans"]:
        assert O.plan_groups(p["n_layers"], p["lp"]) == p["plan"]
    # proj/tests/test_layer_plan.cpp: override grammar and rejections
    assert O.parse_plan("0|1-3|4-6|7") == "0|1-3|4-6|7"
    for bad in ("0|2-3|4", "0|1-3", "0-1|2|3", "", "0||1", "0|3-1|4", "0|x|2"):
        with pytest.raises(O.OracleError):
            O.parse_plan(bad)


def test_tree_commit_then_decode():
    g = NUM["tree_commit"]
    assert len(g["next_logits"]) == 258


@pytest.mark.parametrize("case", GEN, ids=[c["name"] for c in GEN])
def test_generate_matches_reference(case):
    base, draft = _models(case)
    if case["error"] is not None:  # the reference raised (e.g. the greedy sibling CheckError)
        with pytest.raises(O.OracleError, match=case["error"]):
            O.generate(base, draft, _run(case), case["prompt"].encode(), with_cache=False)
        return
    res = O.generate(base, draft, _run(case), case["prompt"].encode(), with_cache=False)
    assert res.tokens == case["tokens"]
    assert len(res.iterations) == len(case["iterations"])
    for it, want in zip(res.iterations, case["iterations"]):
        got = (it.m, it.n, it.drafted_nodes, it.emitted, it.sequential_forwards, it.fuzzy_forwards,
               it.base_forwards, it.committed, it.draft_committed, it.base_committed)
        exp = tuple(want[k] for k in ("m", "n", "drafted_nodes", "emitted", "sequential_forwards",
                                      "fuzzy_forwards", "base_forwards", "committed", "draft_committed",
                                      "base_committed"))
        assert got == exp
        assert np.array_equal(it.draft_kv, np.asarray(want["draft_kv"]))
        assert np.array_equal(it.base_kv, np.asarray(want["base_kv"]))


def test_greedy_chain_kat():
    """proj/tests/test_verifier.cpp:290-318: m=2, tokens [1,0], bonus 2."""
    dists = [[0, 1, 0], [1, 0, 0]]
    base = [[0.1, 0.8, 0.1], [0.9, 0.05, 0.05], [0.2, 0.2, 0.6]]
    m, acc, bonus = O.verify_tree(3, [1, 0], [-1, 0], [0, 1], dists, base, [1, 1], 0.0, 1)
    assert (m, acc, bonus) == (2, [1, 0], 2)


def test_verify_rejects_empty_tree():
    with pytest.raises(O.OracleError) as ei:
        O.verify_tree(1, [], [], [], [[1.0]], [[1.0]], [1], 1.0, 2)
    assert ei.value.kind == "structure"


def test_greedy_multi_sibling_reject_throws_like_reference():
    """proj/src/verifier.cpp:156-157: greedy + width 2 + first sibling rejected."""
    dists = [[0.0, 1.0, 0.0]]
    base = [[1.0, 0.0, 0.0], [1, 0, 0], [1, 0, 0]]
    with pytest.raises(O.OracleError) as ei:
        O.verify_tree(3, [1, 0], [-1, -1], [0, 0], dists, base, [2], 0.0, 1)
    assert ei.value.kind == "check"


def test_width1_chain_rejection_sampling_is_lossless_analytically():
    """One-level induced distribution equals the target (criterion 1 restated
    empirically with the oracle's verify over many seeds)."""
    V = 4
    p = np.array([0.1, 0.2, 0.3, 0.4], np.float32)
    q = np.array([0.4, 0.3, 0.2, 0.1], np.float32)
    counts = np.zeros(V)
    trials = 20000
    for s in range(trials):
        # draw the drafted token with its own stream, verify with another
        u = O.rng_uniforms(s + 1, 1)[0]
        tok = int(np.searchsorted(np.cumsum(q.astype(np.float64)), u, side="right"))
        tok = min(tok, V - 1)
        m, acc, bonus = O.verify_tree(V, [tok], [-1], [0], [q], [p, p], [1], 1.0, 10_000 + s)
        counts[acc[0] if m else bonus] += 1
    assert np.abs(counts / trials - p).max() < 0.015


def test_select_children_topk_ties_and_sampling():
    lg = np.array([1.0, 3.0, 3.0, 2.0], np.float32)
    assert O.select_children(lg, 3, 0.0, 1) == [1, 2, 3]
    picks = O.select_children(lg, 4, 1.0, 7)
    assert sorted(picks) == [0, 1, 2, 3]


def test_config_errors():
    with pytest.raises(O.OracleError) as ei:
        O.Model(O.ModelConfig(d_model=33, n_heads=2, d_head=16))
    assert ei.value.kind == "config"
    base = O.Model(O.tiny_config(4, 101))
    draft = base.truncated(2)
    for run in (O.RunConfig(algorithm="easyspec", n=4, widths=[2, 2, 2, 2], lp_size=2, max_new_tokens=0),
                O.RunConfig(algorithm="sd", n=4, widths=[2, 1, 1, 1], lp_size=2),
                O.RunConfig(algorithm="easyspec", n=4, widths=[2, 2, 2, 2], lp_size=2, max_new_tokens=100000)):
        with pytest.raises(O.OracleError) as ei:
            O.generate(base, draft, run, b"x")
        assert ei.value.kind == "config"
