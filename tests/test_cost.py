"""Cost simulator (proj/src/cost_sim.cpp) through the C
ABI, pinned to fixtures the unmodified reference produced (oracle/ref_dump.cpp
-> tests/golden/ref_cost.json):

* the affine cost model and its compositions, values and error texts — CPU;
* the simulated stage units every generation's traces carry, the SimClock
  occupancy CSV and the report's simulated block and speed-up
  (orchestrator.cpp:72-77, 256-466; report.cpp:51-95) — CPU from the
  reference's own traces, GPU through the engine's generation loop.

Every number is compared with ==: the host arithmetic is double in the
reference's order."""
import json
import os
from dataclasses import replace

import pytest

from paper_2502_02493_b200 import espec as E

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")
COST = json.load(open(os.path.join(GOLD, "ref_cost.json")))
GEN = {c["name"]: c for c in json.load(open(os.path.join(GOLD, "ref_generate.json")))}


def _params(j):
    return E.CostParams(**j)


def test_defaults_are_the_reference_cost_params():
    assert E.cost_defaults() == E.CostParams() == _params(COST["functions"][0]["params"])


@pytest.mark.parametrize("k", range(len(COST["functions"])))
def test_cost_functions_match_reference_bit_for_bit(k):
    f = COST["functions"][k]
    p = _params(f["params"])
    for w, s, tp, want in f["t_exe"]:
        assert E.t_exe(p, w, s, tp) == want
    for g, s, want in f["group_attention"]:
        assert E.group_attention_time(p, g, s) == want
    for plan, s, want in f["draft_group"]:
        if isinstance(want, str):
            with pytest.raises(E.EspecError) as ex:
                E.simulate_draft_group(p, plan, s)
            assert ex.value.kind == "config" and want in str(ex.value)
        else:
            assert E.simulate_draft_group(p, plan, s) == want
    for L, s, want in f["sequential"]:
        assert E.sequential_draft_forward_time(p, L, s) == want
    for L, s, want in f["base"]:
        assert E.base_forward_time(p, L, s) == want
    for L, pl, tk, want in f["vanilla_baseline"]:
        assert E.vanilla_baseline_sim(p, L, pl, tk) == want


def test_total_time_model_and_error_texts_match_reference():
    for n_tok, td, tb, n, alpha, want in COST["total_time"]:
        assert E.total_time_model(n_tok, td, tb, n, alpha) == want
    e = COST["errors"]
    d = E.CostParams()
    cases = [(replace(d, c_mem=-1.0), "negative"), (replace(d, tp_size_base=0), "tp_zero"),
             (replace(d, tp_size_draft=9), "tp_over")]
    for p, key in cases:
        with pytest.raises(E.EspecError) as ex:
            E.cost_validate(p)
        assert ex.value.kind == "config" and e[key] in str(ex.value)
    with pytest.raises(E.EspecError) as ex:
        E.t_exe(d, 0.1, 0.5, 1)
    assert e["t_exe_s"] in str(ex.value)
    with pytest.raises(E.EspecError) as ex:
        E.group_attention_time(d, 0, 1.0)
    assert e["group_zero"] in str(ex.value)
    with pytest.raises(E.EspecError) as ex:
        E.simulate_draft_group(_params(COST["functions"][1]["params"]), "0|1-5|6", 1.0)
    assert e["plan_over"] in str(ex.value)
    with pytest.raises(E.EspecError) as ex:
        E.total_time_model(10, 1, 1, 2, 0.0)
    assert ex.value.kind == "domain" and e["alpha_zero"] in str(ex.value)
    for n, alpha in ((2, 1.5), (0, 0.5)):
        with pytest.raises(E.EspecError) as ex:
            E.total_time_model(10, 1, 1, n, alpha)
        assert ex.value.kind == "config" and e["alpha_over"] in str(ex.value)


RUNS = [r for r in COST["runs"] if r["error"] is None]


def _traces(run, sims):
    out = []
    for it, (c, d, v) in zip(GEN[run["name"]]["iterations"], sims):
        out.append(E.IterationTrace(m=it["m"], n=it["n"], drafted_nodes=it["drafted_nodes"], emitted=it["emitted"],
                                    sequential_forwards=it["sequential_forwards"], fuzzy_forwards=it["fuzzy_forwards"],
                                    base_forwards=it["base_forwards"], committed=0, draft_committed=0,
                                    base_committed=0, bonus=0, calibrate_ms=1.0, draft_ms=1.0, verify_ms=1.0,
                                    calibrate_sim=c, draft_sim=d, verify_sim=v))
    return out


def _check_report(run, traces):
    case = GEN[run["name"]]
    r = E.aggregate(traces, run["vanilla_baseline"])
    assert [r.draft_per_100_sim, r.verify_per_100_sim, r.calibrate_per_100_sim] == run["per100_sim"]
    assert r.draft_total_per_100_sim == run["draft_total_per100_sim"]
    assert r.total_sim == run["total_sim"]
    assert r.speedup_vs_vanilla == run["speedup"]
    rc = case["run"]
    alg = rc["algorithm"]
    csv = E.emit_report(r, traces, alg, 0 if alg == "vanilla" else rc["n"], rc["widths"],
                        rc["lp_size"] if alg == "easyspec" else 1, fmt="csv")
    assert csv == run["csv"]


@pytest.mark.parametrize("run", RUNS, ids=[f"{r['name']}-d{r['cost']['devices']}" for r in RUNS])
def test_report_sim_block_from_reference_traces(run):
    """aggregate / emit_report over the reference's own simulated stage units
    reproduce its report (speed-up, per-100 sim times, CSV) exactly."""
    _check_report(run, _traces(run, run["sims"]))
    p = _params(run["cost"])
    L = GEN[run["name"]]["base"]["n_layers"]
    assert E.vanilla_baseline_sim(p, L, run["prompt_len"], run["n_tokens"]) == run["vanilla_baseline"]


# ---------------------------------------------------------------------------
# GPU: the engine's generation loop advances the same simulated clock
# ---------------------------------------------------------------------------

def _engine(case):
    from tests import test_gpu_parity as G
    return G._engine_for_case(case)


# (the reference's greedy-sibling CheckError fixture is covered by test_gpu_parity)
GPU_RUNS = [r for r in COST["runs"] if r["error"] is None or "devices" in r["error"]]


@pytest.mark.gpu
@pytest.mark.parametrize("run", GPU_RUNS, ids=[f"{r['name']}-d{r['cost']['devices']}" for r in GPU_RUNS])
def test_gpu_generation_sim_units_match_reference(run):
    """Per-iteration calibrate / draft / verify simulated units, the SimClock
    occupancy CSV and the report's simulated block of every generation fixture
    (default cost, and a 4-device cost for three cases) equal the reference's
    bit for bit; a plan wider than the simulated device count fails with the
    reference's ConfigError."""
    case = GEN[run["name"]]
    eng = _engine(case)
    eng.set_cost(_params(run["cost"]))
    if run["error"] is not None:
        with pytest.raises(E.EspecError) as ex:
            eng.generate(case["prompt"].encode())
        assert run["error"] in str(ex.value)
        eng.close()
        return
    toks, traces = eng.generate(case["prompt"].encode())
    assert toks == case["tokens"]
    got = [[t.calibrate_sim, t.draft_sim, t.verify_sim] for t in traces]
    assert got == run["sims"]
    assert eng.occupancy_csv() == run["occupancy"]
    _check_report(run, traces)
    eng.close()
