"""Tensor-parallel path on one B200: all shards of a TP group live in one
process and exchange partial sums through the same one-shot collective
kernels that run over NVLink peer memory between processes (here the peer
pointers are plain device pointers). Checks the sharded math end to end:
every shard emits the same tokens, equal to the reference fixtures (fp32
parity weights, sliced per shard) and, in bf16, greedy speculative == greedy
vanilla within the TP group (fixed rank-order reductions keep it
batch-invariant)."""
import json
import os
from dataclasses import replace

import pytest

from paper_2502_02493_b200 import espec as E

pytestmark = pytest.mark.gpu

GEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "ref_generate.json")))


def _case(name):
    return next(c for c in GEN if c["name"] == name)


def _cfg(j):
    return E.ModelConfig(**{k: j[k] for k in ("vocab_size", "d_model", "n_layers", "n_heads", "d_head", "d_mlp",
                                              "max_positions", "norm_eps", "seed")})


@pytest.mark.parametrize("layout", ["tp", "lp"])  # drafter: tensor-parallel / the paper's layer-parallel placement
@pytest.mark.parametrize("tp", [2])
@pytest.mark.parametrize("idx", [3, 13, 16])  # greedy chain, T=0.8 chain, T=0.8 tree (width 2)
def test_tp_group_matches_reference_fixture(tp, idx, layout):
    case = GEN[idx]
    r = case["run"]
    base = _cfg(case["base"])
    if base.n_heads % tp or base.d_mlp % (16 * tp) or base.vocab_size % tp:
        pytest.skip("shape does not shard")
    run = E.RunConfig(algorithm=r["algorithm"], n=r["n"], widths=r["widths"], lp_size=r["lp_size"],
                      plan_override=r["plan_override"] or None, temperature=r["temperature"],
                      max_new_tokens=r["max_new_tokens"], seed=r["seed"], calibration=r["calibration"])
    assert not case["draft_seed"] and case["keep"] > 0
    engines = E.tp_group_local(base, replace(base, n_layers=case["keep"]), run, tp, truncated=case["keep"],
                               draft_layout=layout)
    outs = E.tp_generate(engines, prompt=case["prompt"].encode())
    for toks, traces in outs:
        assert toks == case["tokens"]
        assert [t.m for t in traces] == [it["m"] for it in case["iterations"]]
    for e in engines:
        e.close()


@pytest.mark.parametrize("layout", ["tp", "lp"])
def test_tp_bf16_greedy_speculative_equals_vanilla(layout):
    base = E.ModelConfig(vocab_size=4096, d_model=512, n_layers=6, n_heads=8, n_kv_heads=2, d_head=64, d_mlp=1536,
                         max_positions=512, seed=5, rope_theta=500000.0, tied_head=False, weight_dtype=E.BF16,
                         kv_dtype=E.BF16)
    draft = replace(base, n_layers=4, seed=105)
    prompt = list(range(7, 40))
    outs = {}
    for alg in ("vanilla", "easyspec"):
        run = E.RunConfig(algorithm=alg, n=5, lp_size=3, temperature=0.0, max_new_tokens=24, seed=1)
        engines = E.tp_group_local(base, draft, run, 2, parity=False, draft_layout=layout)
        res = E.tp_generate(engines, tokens=prompt)
        assert res[0][0] == res[1][0]  # both shards decided the same tokens
        outs[alg] = res[0][0]
        for e in engines:
            e.close()
    assert outs["easyspec"] == outs["vanilla"]


def test_lp_placement_matches_fuzzy_fixtures_with_a_lp4_plan():
    """A 4-layer fuzzy group over 2 ranks: slots 0 and 2 on rank 0, 1 and 3
    on rank 1 (slot j -> rank j mod the group's GPUs), fixture tokens."""
    case = next(c for c in GEN if c["name"] == "fixa_easyspec_lp4")
    r = case["run"]
    base = _cfg(case["base"])
    run = E.RunConfig(algorithm=r["algorithm"], n=r["n"], widths=r["widths"], lp_size=r["lp_size"],
                      temperature=r["temperature"], max_new_tokens=r["max_new_tokens"], seed=r["seed"])
    engines = E.tp_group_local(base, replace(base, n_layers=case["keep"]), run, 2, truncated=case["keep"],
                               draft_layout="lp")
    for toks, traces in E.tp_generate(engines, prompt=case["prompt"].encode()):
        assert toks == case["tokens"]
        assert [t.m for t in traces] == [it["m"] for it in case["iterations"]]
    for e in engines:
        e.close()


def test_lp_layout_config_errors():
    base = E.tiny_config(4, 3)
    run = E.RunConfig(n=2, lp_size=2)
    with pytest.raises(E.EspecError):  # one GPU has no layer-parallel group
        E.Engine(base, replace(base, n_layers=3), run, draft_layout="lp")
    engines = E.tp_group_local(base, replace(base, n_layers=3), run, 2, draft_layout="lp")
    with pytest.raises(E.EspecError) as ex:
        engines[0].share_truncated_draft()
    assert ex.value.kind == "config"
    for e in engines:
        e.close()
