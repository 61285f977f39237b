"""Stage-level C ABI (espec_prefill / calibrate / draft / verify /
resolve_draft_cache / commit_outcome) against the reference's own stage
functions.

tests/golden/ref_stages.json is written by oracle/_ref/ref_dump: the
unmodified reference core re-driven stage by stage through its public
draft_tree (proj/src/draft_engine.cpp:188-289) and verify_tree
(proj/src/verifier.cpp:86-177), pinned against generate() for every case. Each
GPU iteration here is driven through the five stage calls and its DraftTree
and VerificationOutcome must equal the reference's, field for field.
"""
import json
import os
from dataclasses import replace

import numpy as np
import pytest

from paper_2502_02493_b200 import espec as E

from test_gpu_parity import GEN, _engine_for_case, _erun

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
STAGES = {c["name"]: c for c in json.load(open(os.path.join(GOLDEN, "ref_stages.json")))}
CASES = [c for c in GEN if c["name"] in STAGES and STAGES[c["name"]]["error"] is None]


def _prompt_tokens(case):
    return [E.BOS] + list(case["prompt"].encode())


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_stage_api_trees_and_outcomes_match_reference(case):
    ref = STAGES[case["name"]]
    eng = _engine_for_case(case)
    eng.prefill(_prompt_tokens(case))
    out = []
    sampled = case["run"]["temperature"] > 0
    for want in ref["iterations"]:
        eng.calibrate()
        tree = eng.draft(want_dists=sampled)
        wt = want["tree"]
        for k in ("token", "parent", "depth", "prob_index", "cache_row", "first_child", "n_children"):
            assert getattr(tree, k) == wt[k], k
        assert tree.root_children == wt["root_children"]
        assert tree.n_dists == wt["n_dists"]
        if sampled:  # every draft distribution sums to one (fp32 softmax rows)
            np.testing.assert_allclose(tree.dists.astype(np.float64).sum(), wt["dists_sum"], rtol=1e-5)
        o = eng.verify()
        assert (o.m, o.n, o.path, o.tokens, o.bonus) == (want["m"], want["n"], want["path"], want["accepted"],
                                                         want["bonus"])
        eng.resolve_draft_cache(o)
        em, tr = eng.commit_outcome()
        assert (tr.draft_committed, tr.base_committed) == (want["draft_committed"], want["base_committed"])
        out += em
    assert out == ref["tokens"]
    assert eng.done()
    eng.close()


def test_stage_api_equals_fused_step_bf16():
    """The five stage calls and espec_step run the same kernels: a bf16 GQA
    pair yields bitwise-identical emitted tokens and traces either way."""
    base = E.ModelConfig(vocab_size=4096, d_model=512, n_layers=6, n_heads=8, n_kv_heads=2, d_head=64, d_mlp=1536,
                         max_positions=1024, seed=5, weight_dtype=E.BF16, kv_dtype=E.BF16, tied_head=False,
                         rope_theta=500000.0)
    draft = replace(base, n_layers=4, seed=9)
    run = E.RunConfig(algorithm="easyspec", n=4, widths=[2, 2, 1, 1], lp_size=2, temperature=0.0,
                      max_new_tokens=32, seed=1)
    prompt = list(np.random.default_rng(3).integers(0, 4096, 300))
    res = []
    for staged in (False, True):
        eng = E.Engine(base, draft, run)
        eng.init_weights(E.Engine.BASE, base.seed, parity=False)
        eng.init_weights(E.Engine.DRAFT, draft.seed, parity=False)
        toks, ms = [], []
        if staged:
            eng.prefill(prompt)
            while not eng.done():
                em, tr, _, _ = eng.iterate_stages()
                toks += em
                ms.append(tr.m)
        else:
            eng.begin(prompt)
            while not eng.done():
                em, tr = eng.step()
                toks += em
                ms.append(tr.m)
        res.append((toks, ms))
        eng.close()
    assert res[0] == res[1]


def test_verify_accepts_a_caller_tree_of_the_base_continuation():
    """verify_tree on a caller-edited tree (verifier.hpp:51-52): replacing a
    chain's tokens by the base model's own greedy continuation makes every
    level accept (m = n) and the bonus the next greedy token."""
    case = next(c for c in GEN if c["name"] == "indep_greedy_easyspec")
    van = next(c for c in GEN if c["name"] == "indep_greedy_vanilla")
    eng = _engine_for_case(case)
    n = case["run"]["n"]
    eng.prefill(_prompt_tokens(case))
    greedy = van["tokens"]
    emitted = []
    for it in range(3):
        def edit(tree):
            start = len(emitted)
            for j in range(len(tree.token)):  # chain: node j at depth j + 1
                tree.token[j] = greedy[start + j]
        em, tr, tree, o = eng.iterate_stages(edit)
        assert o.m == n and o.tokens == greedy[len(emitted): len(emitted) + n]
        assert o.bonus == greedy[len(emitted) + n]
        emitted += em
    assert emitted == greedy[: len(emitted)]
    eng.close()


def test_stage_order_is_enforced():
    case = next(c for c in GEN if c["name"] == "indep_greedy_easyspec")
    eng = _engine_for_case(case)
    eng.prefill(_prompt_tokens(case))
    with pytest.raises(E.EspecError) as ex:
        eng.verify()
    assert ex.value.kind == "structure"
    eng.calibrate()
    with pytest.raises(E.EspecError):
        eng.calibrate()
    tree = eng.draft()
    tree.parent[-1] = -1  # a different shape than drafted
    with pytest.raises(E.EspecError) as ex:
        eng.verify(tree)
    assert ex.value.kind == "structure"
    eng.close()


def test_greedy_sibling_rejection_reference_error_and_default_rule():
    """The fixture where the reference raises CheckError('sibling candidates
    exhaust the draft distribution', verifier.cpp:146-158): strict mode raises
    the same error through the C ABI; the default rule accepts the sibling
    equal to the base argmax and stays lossless (equals greedy vanilla)."""
    case = next(c for c in GEN if c["name"] == "greedy_tree_throws_indep")
    van = next(c for c in GEN if c["name"] == "indep_greedy_vanilla")
    assert case["error"] == "sibling candidates exhaust the draft distribution"
    eng = _engine_for_case(case)
    eng.set_run(_erun(case, strict_greedy_tree=True))
    with pytest.raises(E.EspecError) as ex:
        eng.generate(case["prompt"].encode())
    assert ex.value.kind == "check" and case["error"] in str(ex.value)
    eng.set_run(_erun(case))
    toks, traces = eng.generate(case["prompt"].encode())
    assert toks == van["tokens"][: len(toks)] and len(toks) == case["run"]["max_new_tokens"]
    assert any(t.m < t.n for t in traces)
    eng.close()
