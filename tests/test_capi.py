"""C-ABI boundary checks that need no GPU: the library loads, exports every
symbol include/espec_c.h declares, and its host-side logic (layer plans,
config validation) matches the reference."""
import ctypes
import json
import os
import re

import pytest

from paper_2502_02493_b200 import espec as E

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "espec_c.h")).read()
    return sorted(set(re.findall(r"\b(espec_[a-z_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(E.LIB_PATH)
    names = _declared()
    assert len(names) >= 20
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_library_is_sm100a():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", E.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_plans_match_reference_goldens():
    golden = json.load(open(os.path.join(ROOT, "tests", "golden", "ref_numerics.json")))
    for p in golden["plans"]:
        assert E.plan_groups(p["n_layers"], p["lp"]) == p["plan"]
    assert E.parse_plan_override("0|1-3|4-6|7") == "0|1-3|4-6|7"
    for bad in ("0|2-3|4", "0|1-3", "0-1|2|3", "0||1", "0|3-1|4", "0|x|2", "0|1|"):
        with pytest.raises(E.EspecError) as ei:
            E.parse_plan_override(bad)
        assert ei.value.kind == "config"


@pytest.mark.parametrize("bad", [dict(d_model=33, n_heads=2, d_head=16), dict(n_layers=1), dict(d_head=15),
                                 dict(vocab_size=1), dict(n_heads=4, n_kv_heads=3)])
def test_model_config_validation(bad):
    cfg = E.ModelConfig(**{**E.tiny_config(4, 1).__dict__, **bad})
    with pytest.raises(E.EspecError) as ei:
        E.Engine(cfg, E.tiny_config(2, 1), E.RunConfig(n=4, lp_size=2))
    assert ei.value.kind == "config"


def test_run_config_validation():
    b, d = E.tiny_config(4, 1), E.tiny_config(2, 1)
    for run in (E.RunConfig(algorithm="sd", n=4, widths=[2, 1, 1, 1]), E.RunConfig(n=4, widths=[2, 2]),
                E.RunConfig(n=4, max_new_tokens=0), E.RunConfig(n=0)):
        with pytest.raises(E.EspecError) as ei:
            E.Engine(b, d, run)
        assert ei.value.kind == "config"


def test_vocab_mismatch_rejected():
    with pytest.raises(E.EspecError) as ei:
        E.Engine(E.tiny_config(4, 1), E.ModelConfig(vocab_size=300, d_model=32, n_heads=2, d_head=16, d_mlp=64,
                                                     n_layers=2), E.RunConfig(n=4, lp_size=2))
    assert ei.value.kind == "config"


def test_total_variation_matches_definition():
    """espec_total_variation = total_variation (proj/src/orchestrator.cpp:
    528-553) on the reference's own criterion-2 prefix counts."""
    golden = json.load(open(os.path.join(ROOT, "tests", "golden", "ref_prefix.json")))
    runs = golden["runs"]
    a = {tuple(e["prefix"]): e["count"] for e in golden["easyspec"]}
    b = {tuple(e["prefix"]): e["count"] for e in golden["vanilla"]}
    keys = set(a) | set(b)
    want = 0.5 * sum(abs(a.get(k, 0) - b.get(k, 0)) / runs for k in keys)
    assert abs(E.total_variation(a, b, runs, runs) - want) < 1e-12
    assert E.total_variation(a, a, runs, runs) == 0.0
