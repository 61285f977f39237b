"""GPU parity: the sm_100a engine (through the C ABI) against the CPU oracle
and the reference's golden fixtures.

Bars (stated per test):
  * fp32 parity mode: weights bit-identical to init_model; logits / hidden /
    K/V within 2e-4 absolute (+1e-4 relative) of the oracle (different fp32
    summation order; the reference itself is the 1-ulp-per-op oracle);
    emitted token ids, accepted counts m, cache lengths and forward counts
    bit-exact against the reference fixtures.
  * bf16 perf mode: logits within 2e-2 (+2e-2 rel) of a PyTorch fp32
    restatement on the same (bf16-rounded) weights; greedy EasySpec /
    SD output identical to vanilla greedy (losslessness, batch invariance).
"""
import json
import os
from dataclasses import replace

import numpy as np
import pytest

from oracle import oracle as O
from paper_2502_02493_b200 import espec as E

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
NUM = json.load(open(os.path.join(GOLDEN, "ref_numerics.json")))
GEN = json.load(open(os.path.join(GOLDEN, "ref_generate.json")))
FP32_ATOL, FP32_RTOL = 2e-4, 1e-4


def _ecfg(j, **kw):
    c = E.ModelConfig(**{k: j[k] for k in ("vocab_size", "d_model", "n_layers", "n_heads", "d_head", "d_mlp",
                                           "max_positions", "norm_eps", "seed")})
    return replace(c, **kw)


def _ocfg(j):
    return O.ModelConfig(**{k: j[k] for k in ("vocab_size", "d_model", "n_layers", "n_heads", "d_head", "d_mlp",
                                               "max_positions", "norm_eps", "seed")})


def _erun(case, **kw):
    r = case["run"]
    run = E.RunConfig(algorithm=r["algorithm"], n=r["n"], widths=r["widths"], lp_size=r["lp_size"],
                      plan_override=r["plan_override"] or None, temperature=r["temperature"],
                      max_new_tokens=r["max_new_tokens"], seed=r["seed"], calibration=r["calibration"])
    return replace(run, **kw)


def _engine_for_case(case):
    base = _ecfg(case["base"])
    run = _erun(case)
    if case["draft_seed"]:
        d = replace(base, n_layers=case["keep"], seed=case["draft_seed"])
        eng = E.Engine(base, d, run)
        eng.init_weights(E.Engine.BASE, base.seed)
        eng.init_weights(E.Engine.DRAFT, d.seed)
        return eng
    if case["keep"] == 0:  # self-drafting: an identical independent copy
        eng = E.Engine(base, base, run)
        eng.init_weights(E.Engine.BASE, base.seed)
        eng.init_weights(E.Engine.DRAFT, base.seed)
        return eng
    return E.truncated_pair(base, case["keep"], run)


def _close(a, b, atol=FP32_ATOL, rtol=FP32_RTOL):
    np.testing.assert_allclose(a, b, atol=atol, rtol=rtol)


def test_parity_init_weights_bit_identical():
    cfg = E.tiny_config(3, 99)
    eng = E.Engine(cfg, replace(cfg, n_layers=2), E.RunConfig(n=4, lp_size=2))
    eng.init_weights(E.Engine.BASE, 99)
    om = O.Model(O.tiny_config(3, 99))
    d, f = cfg.d_model, cfg.d_mlp
    assert np.array_equal(eng.read_tensor(1, "embedding", cfg.vocab_size, d), om.tensor("embedding"))
    for layer in range(3):
        for name, shape in (("wq", (d, d)), ("wk", (d, d)), ("wv", (d, d)), ("wo", (d, d)), ("w_gate", (d, f)),
                            ("w_up", (d, f)), ("w_down", (f, d))):
            assert np.array_equal(eng.read_tensor(1, name, *shape, layer=layer), om.tensor(name, layer)), name


def test_golden_argmax_110_and_logits():
    g = NUM["golden_argmax"]
    cfg = _ecfg(g["config"])
    eng = E.Engine(cfg, replace(cfg, n_layers=2), E.RunConfig(n=4, lp_size=2))
    eng.init_weights(E.Engine.BASE, cfg.seed)
    logits, _ = eng.forward(E.Engine.BASE, E.tokenize(b"golden"))
    assert int(np.argmax(logits[-1])) == 110
    _close(logits[-1], np.asarray(g["logits"], np.float32))


def test_prefill_hidden_logits_kv_vs_oracle():
    g = NUM["prefill_kv"]
    cfg = _ecfg(g["config"])
    eng = E.Engine(cfg, cfg, E.RunConfig(n=4, lp_size=1))
    eng.init_weights(E.Engine.BASE, cfg.seed)
    logits, hidden = eng.forward(E.Engine.BASE, E.tokenize(b"ab"))
    _close(hidden.ravel(), np.asarray(g["hidden"], np.float32))
    _close(logits.ravel(), np.asarray(g["logits"], np.float32))
    for layer in range(2):
        k, v, n = eng.cache_view(E.Engine.BASE, layer)
        assert n == 3
        _close(k.ravel(), np.asarray(g["kv"][layer]["k"], np.float32))
        _close(v.ravel(), np.asarray(g["kv"][layer]["v"], np.float32))


@pytest.mark.parametrize("lp", [1, 2, 3, 4])
def test_fuzzy_forward_vs_reference(lp):
    g = NUM["fuzzy"]
    cfg = _ecfg(g["config"])
    eng = E.Engine(cfg, cfg, E.RunConfig(n=4, lp_size=lp))
    eng.init_weights(E.Engine.DRAFT, cfg.seed)
    logits, hidden = eng.forward(E.Engine.DRAFT, g["tokens"], plan=f"lp={lp}")
    _close(hidden.ravel(), np.asarray(g[f"lp{lp}"]["hidden"], np.float32))
    _close(logits.ravel(), np.asarray(g[f"lp{lp}"]["logits"], np.float32))


def test_all_singleton_fuzzy_equals_sequential_bitwise():
    """Criterion 3 (proj/tests/acceptance_main.cpp:186-217) on device."""
    cfg = E.tiny_config(6, 63)
    eng = E.Engine(cfg, cfg, E.RunConfig(n=4, lp_size=1))
    eng.init_weights(E.Engine.DRAFT, 63)
    rng = np.random.default_rng(64)
    for _ in range(8):
        toks = [int(t) for t in rng.integers(0, 256, size=int(rng.integers(1, 6)))]
        a = eng.forward(E.Engine.DRAFT, toks, plan="lp=1")
        b = eng.forward(E.Engine.DRAFT, toks)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


# fixtures where the reference raised are covered in test_gpu_stages.py
GREEDY_CHAINS = [c for c in GEN if c["error"] is None and c["run"]["temperature"] == 0.0
                 and max(c["run"]["widths"]) == 1]


@pytest.mark.parametrize("case", GREEDY_CHAINS, ids=[c["name"] for c in GREEDY_CHAINS])
def test_generate_matches_reference_tokens(case):
    """Emitted tokens, m per iteration, cache lengths and forward counts are
    bit-exact against the reference; K/V checksums within fp32 tolerance."""
    eng = _engine_for_case(case)
    toks, traces = eng.generate(case["prompt"].encode())
    assert toks == case["tokens"]
    assert len(traces) == len(case["iterations"])
    for t, want in zip(traces, case["iterations"]):
        assert (t.m, t.emitted, t.drafted_nodes, t.sequential_forwards, t.fuzzy_forwards, t.base_forwards,
                t.committed, t.draft_committed, t.base_committed) == \
               (want["m"], want["emitted"], want["drafted_nodes"], want["sequential_forwards"],
                want["fuzzy_forwards"], want["base_forwards"], want["committed"], want["draft_committed"],
                want["base_committed"])
    last = case["iterations"][-1]
    for which, key in ((E.Engine.DRAFT, "draft_kv"), (E.Engine.BASE, "base_kv")):
        cfg = eng.draft_cfg if which == E.Engine.DRAFT else eng.base_cfg
        for layer in range(cfg.n_layers):
            k, v, n = eng.cache_view(which, layer)
            got = [k.astype(np.float64).sum(), np.abs(k).astype(np.float64).sum(), v.astype(np.float64).sum(),
                   np.abs(v).astype(np.float64).sum()]
            np.testing.assert_allclose(got, last[key][layer], rtol=1e-4, atol=1e-2 * max(1, n))


SAMPLED_OR_TREES = [c for c in GEN if c not in GREEDY_CHAINS and c["error"] is None]


@pytest.mark.parametrize("case", SAMPLED_OR_TREES, ids=[c["name"] for c in SAMPLED_OR_TREES])
def test_generate_sampled_and_trees_match_reference(case):
    """T > 0 rejection sampling (uniforms drawn from the reference's xoshiro
    stream in the reference's order) and multi-sibling tree levels
    (top-k at T = 0): emitted tokens, m, drafted nodes, forward counts and
    cache lengths bit-exact against the reference fixtures."""
    eng = _engine_for_case(case)
    toks, traces = eng.generate(case["prompt"].encode())
    assert toks == case["tokens"]
    assert len(traces) == len(case["iterations"])
    for t, want in zip(traces, case["iterations"]):
        assert (t.m, t.emitted, t.drafted_nodes, t.sequential_forwards, t.fuzzy_forwards, t.base_forwards,
                t.committed, t.draft_committed, t.base_committed) == \
               (want["m"], want["emitted"], want["drafted_nodes"], want["sequential_forwards"],
                want["fuzzy_forwards"], want["base_forwards"], want["committed"], want["draft_committed"],
                want["base_committed"])


PREFIX = json.load(open(os.path.join(GOLDEN, "ref_prefix.json")))


def _crit2_engine(alg):
    """Acceptance criterion 2's pair and run (proj/tests/acceptance_main.cpp:156-183)."""
    base = E.tiny_config(4, 21, max_positions=64)
    run = E.RunConfig(algorithm=alg, n=3, widths=[2, 2, 2], lp_size=2, temperature=0.8, max_new_tokens=2, seed=11)
    return E.truncated_pair(base, 3, run)


@pytest.mark.parametrize("alg", ["easyspec", "vanilla"])
def test_prefix_distribution_matches_reference_counts(alg):
    """prefix_distribution (orchestrator.cpp:494-526) on device: the same
    per-run seeds give the reference's exact counts for every 2-token prefix
    over 2000 runs (bit-exact sampling, not just the same law)."""
    want = {tuple(e["prefix"]): e["count"] for e in PREFIX[alg]}
    eng = _crit2_engine(alg)
    assert eng.prefix_distribution(b"easyspec", PREFIX["runs"]) == want
    eng.close()
    engines = [_crit2_engine(alg) for _ in range(3)]  # threaded split: same counts
    assert E.prefix_distribution(engines, b"easyspec", PREFIX["runs"]) == want
    for e in engines:
        e.close()


def test_statistical_losslessness_criterion_2():
    """Acceptance criterion 2 at full strength (proj/tests/acceptance_main.cpp:
    156-183): T = 0.8 EasySpec with a [2,2,2] tree vs vanilla, first 2
    tokens, 2 x 200k runs, TV < 0.01."""
    runs = 200_000
    dist = {}
    for alg in ("easyspec", "vanilla"):
        engines = [_crit2_engine(alg) for _ in range(4)]  # 4 host threads, as the reference's threads
        dist[alg] = E.prefix_distribution(engines, b"easyspec", runs)
        for e in engines:
            e.close()
    tv = E.total_variation(dist["easyspec"], dist["vanilla"], runs, runs)
    print(f"criterion 2: TV(easyspec, vanilla) = {tv:.5f} over 2 x {runs} runs, "
          f"{len(dist['easyspec'])}/{len(dist['vanilla'])} distinct prefixes")
    assert tv < 0.01, tv


def test_calibrated_drafter_cache_equals_fresh_prefill_every_iteration():
    """Criterion 4 (proj/tests/acceptance_main.cpp:221-275) / test_orchestrator
    144-177: after each calibrated iteration the drafter cache holds exactly
    the precise K/V of the committed prefix (no fuzzy rows survive)."""
    base = E.tiny_config(8, 21, max_positions=256)
    run = E.RunConfig(algorithm="easyspec", n=4, lp_size=3, temperature=0.0, max_new_tokens=30, seed=1)
    eng = E.truncated_pair(base, 6, run)
    ob = O.Model(O.tiny_config(8, 21, max_positions=256))
    od = ob.truncated(6)
    eng.begin(E.tokenize(b"calibration check"))
    iters = 0
    while not eng.done():
        eng.step()
        committed = eng.committed()
        _, _, covered = eng.cache_view(E.Engine.DRAFT, 0, 0, 0)
        assert 0 < covered <= len(committed)
        _, _, k_ref, v_ref = od.prefill(committed[:covered])
        for layer in range(6):
            k, v, _ = eng.cache_view(E.Engine.DRAFT, layer)
            _close(k, k_ref[layer])
            _close(v, v_ref[layer])
        iters += 1
    assert iters >= 3


def test_greedy_speculative_equals_vanilla_independent_drafter_fp32():
    """Losslessness with rejections: independent drafter (alpha ~ 0)."""
    base = E.tiny_config(8, 11, d_model=64, n_heads=4, d_head=16, d_mlp=128, max_positions=256)
    d = replace(base, n_layers=5, seed=9)
    outs = {}
    for alg in ("vanilla", "sd", "easyspec"):
        eng = E.Engine(base, d, E.RunConfig(algorithm=alg, n=5, lp_size=4, max_new_tokens=40))
        eng.init_weights(E.Engine.BASE, base.seed)
        eng.init_weights(E.Engine.DRAFT, d.seed)
        outs[alg], _ = eng.generate(b"independent")
    assert outs["sd"] == outs["vanilla"] == outs["easyspec"]


def _bf16_pair(d_model=512, n_layers=6, keep=4, n_heads=8, n_kv=2, dh=64, f=1536, vocab=4096, seed=5):
    base = E.ModelConfig(vocab_size=vocab, d_model=d_model, n_layers=n_layers, n_heads=n_heads, n_kv_heads=n_kv,
                         d_head=dh, d_mlp=f, max_positions=1024, seed=seed, rope_theta=500000.0,
                         tied_head=False, weight_dtype=E.BF16, kv_dtype=E.BF16)
    return base, replace(base, n_layers=keep, seed=seed + 100)


def _weights(eng, which, cfg):
    import torch
    d, H, Hkv, dh, f, V = cfg.d_model, cfg.n_heads, cfg.n_kv_heads, cfg.d_head, cfg.d_mlp, cfg.vocab_size
    W = {"embedding": eng.read_tensor(which, "embedding", V, d), "head": eng.read_tensor(which, "head", d, V),
         "final_norm_gain": eng.read_tensor(which, "final_norm_gain", 1, d)[0]}
    for l in range(cfg.n_layers):
        for name, shape in (("wq", (d, H * dh)), ("wk", (d, Hkv * dh)), ("wv", (d, Hkv * dh)), ("wo", (H * dh, d)),
                            ("w_gate", (d, f)), ("w_up", (d, f)), ("w_down", (f, d))):
            W[f"{name}.{l}"] = eng.read_tensor(which, name, *shape, layer=l)
        W[f"attn_norm_gain.{l}"] = np.ones(d, np.float32)
        W[f"mlp_norm_gain.{l}"] = np.ones(d, np.float32)
    return {k: torch.from_numpy(np.ascontiguousarray(v)) for k, v in W.items()}


def test_bf16_forward_matches_torch_fp32_reference():
    from tests import torch_ref
    base, draft = _bf16_pair()
    eng = E.Engine(base, draft, E.RunConfig(n=5, lp_size=2))
    eng.init_weights(E.Engine.BASE, base.seed, parity=False)
    eng.init_weights(E.Engine.DRAFT, draft.seed, parity=False)
    rng = np.random.default_rng(3)
    toks = [int(t) for t in rng.integers(0, base.vocab_size, size=40)]
    for which, cfg, plan in ((E.Engine.BASE, base, None), (E.Engine.DRAFT, draft, None),
                             (E.Engine.DRAFT, draft, "lp=2")):
        logits, hidden = eng.forward(which, toks, plan=plan)
        W = _weights(eng, which, cfg)
        groups = None
        if plan:
            groups = [[int(x) for x in range(int(g.split("-")[0]), int(g.split("-")[-1]) + 1)]
                      for g in E.plan_groups(cfg.n_layers, 2).split("|")]
        ref_logits, ref_hidden = torch_ref.forward(W, cfg, toks, groups)
        scale = float(np.abs(ref_logits.numpy()).max())
        np.testing.assert_allclose(logits, ref_logits.numpy(), atol=2e-2 * scale, rtol=2e-2)
        assert (np.argmax(logits, -1) == ref_logits.numpy().argmax(-1)).mean() > 0.9


def test_bf16_greedy_easyspec_and_sd_equal_vanilla():
    """Greedy losslessness on the perf path: draft/verify batch shapes differ
    (T=1 drafts, T=n+1 verify), outputs must not."""
    base, draft = _bf16_pair()
    outs = {}
    for alg in ("vanilla", "sd", "easyspec"):
        eng = E.Engine(base, draft, E.RunConfig(algorithm=alg, n=5, lp_size=2, max_new_tokens=48))
        eng.init_weights(E.Engine.BASE, base.seed, parity=False)
        eng.init_weights(E.Engine.DRAFT, draft.seed, parity=False)
        outs[alg], traces = eng.generate(bytes(range(32, 96)))
        eng.close()
    assert outs["vanilla"] == outs["sd"] == outs["easyspec"]


def test_bf16_truncated_drafter_accepts_and_is_lossless():
    base, _ = _bf16_pair(n_layers=8)
    outs, alphas = {}, {}
    for alg in ("vanilla", "easyspec"):
        run = E.RunConfig(algorithm=alg, n=5, lp_size=3, max_new_tokens=64)
        eng = E.truncated_pair(base, 6, run, parity=False)
        outs[alg], traces = eng.generate(b"truncated drafter")
        att = sum(t.n for t in traces)
        alphas[alg] = sum(t.m for t in traces) / att if att else 0
        eng.close()
    assert outs["vanilla"] == outs["easyspec"]
    assert alphas["easyspec"] > 0.0  # random-init pair: any acceptance exercises the accept path


def test_bf16_rows_bitwise_independent_of_pass_size():
    """Batch invariance across the decode-GEMV variants: the
    logits of row t are bit-identical whether it is the last row of a (t+1)-row
    pass (8-row variant for t < 8) or one row of a 16-row pass (16-row variant,
    3 epilogue warps), for the base model's (K, N)-only plan."""
    base, draft = _bf16_pair()
    eng = E.Engine(base, draft, E.RunConfig(n=5, lp_size=2))
    eng.init_weights(E.Engine.BASE, base.seed, parity=False)
    eng.init_weights(E.Engine.DRAFT, draft.seed, parity=False)
    rng = np.random.default_rng(17)
    toks = [int(t) for t in rng.integers(0, base.vocab_size, size=16)]
    full, hfull = eng.forward(E.Engine.BASE, toks)
    for t in (0, 3, 7, 8, 12, 15):
        part, hpart = eng.forward(E.Engine.BASE, toks[: t + 1])
        assert np.array_equal(part[t], full[t]), t
        assert np.array_equal(hpart[t], hfull[t]), t
    eng.close()


@pytest.mark.parametrize("widths,n", [([3, 2, 1], 3), (None, 8)])
def test_bf16_greedy_trees_and_long_chains_equal_vanilla(widths, n):
    """Greedy losslessness when the verify pass leaves the 8-row GEMV variant:
    a [3,2,1] tree (16 verify rows) and an n = 8 chain (9 rows)."""
    base, draft = _bf16_pair()
    outs = {}
    for alg in ("vanilla", "easyspec"):
        run = E.RunConfig(algorithm=alg, n=n if alg != "vanilla" else 5, widths=widths if alg != "vanilla" else None,
                          lp_size=2, max_new_tokens=40)
        eng = E.Engine(base, draft, run)
        eng.init_weights(E.Engine.BASE, base.seed, parity=False)
        eng.init_weights(E.Engine.DRAFT, draft.seed, parity=False)
        outs[alg], _ = eng.generate(bytes(range(40, 100)))
        eng.close()
    assert outs["vanilla"] == outs["easyspec"]


@pytest.mark.parametrize("K,N", [(512, 1536), (4096, 4096), (28672, 8192)])
def test_decode_gemv_row_bitwise_independent_of_rows(K, N):
    """espec_probe_gemv: row 0 of the decode GEMV is bit-identical for every
    pass size T = 1..16 (8-row and 16-row kernel variants, any epilogue-warp
    count), for the store and residual epilogues."""
    import ctypes as C
    L = E.lib()
    F = C.POINTER(C.c_float)
    L.espec_probe_gemv.argtypes = [C.c_int] * 4 + [F, F, F, C.c_int]
    rng = np.random.default_rng(K + N)
    x = rng.standard_normal((16, K)).astype(np.float32)
    w = (rng.standard_normal((K, N)) * 0.02).astype(np.float32)
    ref = None
    for T in (1, 2, 5, 8, 9, 12, 13, 16):
        for epi in (0, 1):
            out = np.zeros((T, N), np.float32)
            assert L.espec_probe_gemv(T, K, N, epi, x.ctypes.data_as(F), w.ctypes.data_as(F),
                                      out.ctypes.data_as(F), 0) == 0
            if ref is None:
                ref = out[0].copy()
            assert np.array_equal(out[0], ref), (T, epi)


def test_decode_gemv_row_bitwise_pair_aligned_ranges():
    """The 8192 x 10240 (base QKV) shape takes pair-aligned one-slot CTA ranges
    at 11-16 pass rows (gemv_stream.cu launch_sgemv) and balanced two-slot
    ranges at 9-10, 8-row kernels below: row 0 must stay bit-identical."""
    import ctypes as C
    L = E.lib()
    F = C.POINTER(C.c_float)
    L.espec_probe_gemv.argtypes = [C.c_int] * 4 + [F, F, F, C.c_int]
    K, N = 8192, 10240
    rng = np.random.default_rng(7)
    x = rng.standard_normal((16, K)).astype(np.float32)
    w = (rng.standard_normal((K, N)) * 0.02).astype(np.float32)
    ref = None
    for T in (1, 8, 9, 12, 16):
        for epi in (0, 1):
            out = np.zeros((T, N), np.float32)
            assert L.espec_probe_gemv(T, K, N, epi, x.ctypes.data_as(F), w.ctypes.data_as(F),
                                      out.ctypes.data_as(F), 0) == 0
            if ref is None:
                ref = out[0].copy()
            assert np.array_equal(out[0], ref), (T, epi)


@pytest.mark.parametrize("switch", ["ESPEC_FUSE_ADDS", "ESPEC_B16_ACTS"])
@pytest.mark.parametrize("T", [1, 4, 13])
def test_bf16_decode_fusions_bitwise_equal_unfused(switch, T):
    """Fuzzy groups fold h += attn_i into the O / down GEMV epilogues, and decode
    passes keep the attention / SiLU outputs in bf16 for the O / down GEMVs; both
    must be bit-identical to the unfused path (the switch set to 0)."""
    base, draft = _bf16_pair()
    rng = np.random.default_rng(T)
    toks = [int(t) for t in rng.integers(0, base.vocab_size, size=T)]
    res = {}
    for on in ("1", "0"):
        os.environ[switch] = on
        try:
            eng = E.Engine(base, draft, E.RunConfig(n=5, lp_size=2))
        finally:
            os.environ.pop(switch, None)
        eng.init_weights(E.Engine.BASE, base.seed, parity=False)
        eng.init_weights(E.Engine.DRAFT, draft.seed, parity=False)
        res[on] = [eng.forward(E.Engine.DRAFT, toks, plan=p) for p in ("lp=2", "lp=3")]
        res[on].append(eng.forward(E.Engine.BASE, toks))
        eng.close()
    for (la, ha), (lb, hb) in zip(res["1"], res["0"]):
        assert np.array_equal(la, lb) and np.array_equal(ha, hb)


_POOL_PROBE = r"""
import sys, hashlib, ctypes as C, numpy as np
sys.path.insert(0, sys.argv[1])
from paper_2502_02493_b200 import espec as E
L = E.lib(); F = C.POINTER(C.c_float)
L.espec_probe_gemv.argtypes = [C.c_int] * 4 + [F, F, F, C.c_int]
h = hashlib.sha256()
for K, N, T in ((8192, 10240, 6), (4096, 14336, 1), (28672, 8192, 8), (8192, 8192, 13)):
    rng = np.random.default_rng(K + N + T)
    x = rng.standard_normal((16, K)).astype(np.float32)
    w = (rng.standard_normal((K, N)) * 0.02).astype(np.float32)
    for epi in (0, 1):
        out = np.zeros((T, N), np.float32)
        assert L.espec_probe_gemv(T, K, N, epi, x.ctypes.data_as(F), w.ctypes.data_as(F), out.ctypes.data_as(F), 0) == 0
        h.update(out.tobytes())
print(h.hexdigest())
"""


def test_decode_gemv_tail_pool_bitwise_equal_static():
    """The tail pool hands the last groups of every (problem, k-chunk) pair to
    whichever CTA claims them first; outputs must be bit-identical to fully
    static ranges (ESPEC_SG_POOL=0) — run in fresh processes, as the switch is
    read once per process."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    digests = {}
    for pct in ("0", "12", "30"):
        env = dict(os.environ, ESPEC_SG_POOL=pct)
        r = subprocess.run([sys.executable, "-c", _POOL_PROBE, root], env=env, capture_output=True, text=True,
                           timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        digests[pct] = r.stdout.strip().splitlines()[-1]
    assert digests["0"] == digests["12"] == digests["30"], digests
