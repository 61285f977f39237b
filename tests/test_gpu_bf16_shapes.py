"""bf16 perf kernels at the BASELINE.json shapes against an fp64 reference.

The kernels behind every bench number — the stream-K decode GEMV
(sgemv_kernel: split-K, tail pool, 8-/16-row variants, pair-aligned ranges),
the split-KV tensor-core attention (attn_mma_kernel, tree mask), the fused
RMSNorm / RoPE / SiLU / residual epilogues and the tcgen05 prompt prefill
(tc_gemm_kernel) — run on 2-4-layer models with the EXACT widths of
BASELINE configs[1..3] (C2 Llama-3-70B/8B, C3 Qwen2-72B/7B, C4
Qwen2.5-32B/0.5B; GQA, untied head, rope base, full vocabularies). Each
probe prefills a 2100-row context (several split-KV chunks) through the
tcgen05 prefill, then runs ONE decode-sized pass over a tree of T rows
(T = 1, 6, 9, 16: the chain and [2,2,1] / [3,2,1] verify shapes; 37 rows for
the two-pass > 16-row path) — espec_forward_tree.

Reference: tests/torch_ref.py (pinned to the reference's golden vectors by
test_torch_ref.py) in fp64 on the GPU, on the engine's own bf16 weights read
back through espec_read_tensor.

Stated bound, per row of logits and of final hidden state:
  ||got - ref||_2 <= 1e-2 ||ref||_2   and   max |got - ref| <= 5e-2 RMS(ref),
argmax equal on every row whose reference top-2 margin exceeds 2 x 5e-2 RMS.
Why: the engine stores K/V and feeds every GEMV / MMA with bf16 operands
(relative rounding 2^-9 per element, at ~6 points per layer) and accumulates
in fp32 on the tensor cores; measured over C2/C3/C4 x {base, fuzzy drafter}
x T = 1..16 the worst rows are 0.69 % (L2) and 3.6 % (max), with no
dependence on T, the pass variant or the shape (profiles/r2_bf16_parity.txt).
A fp64 reference that also rounds at the engine's points is no closer
(tools/diag_bf16.py): the residual is bf16 rounding-boundary flips driven by
the tensor-core accumulation order, not a kernel defect. A rotary off-by-one
(the negative control in the test) lands > 5x outside the L2 bound.
"""
import os
import subprocess
import sys
from dataclasses import replace
from types import SimpleNamespace

import numpy as np
import pytest

from paper_2502_02493_b200 import espec as E

pytestmark = pytest.mark.gpu

BOUND_L2, BOUND_MAX = 1e-2, 5e-2
CTX = 2100

C2_BASE = dict(vocab_size=128256, d_model=8192, n_heads=64, n_kv_heads=8, d_head=128, d_mlp=28672,
               rope_theta=500000.0)
C2_DRAFT = dict(vocab_size=128256, d_model=4096, n_heads=32, n_kv_heads=8, d_head=128, d_mlp=14336,
                rope_theta=500000.0)
C3_BASE = dict(vocab_size=152064, d_model=8192, n_heads=64, n_kv_heads=8, d_head=128, d_mlp=29568,
               rope_theta=1000000.0)
C3_DRAFT = dict(vocab_size=152064, d_model=3584, n_heads=28, n_kv_heads=4, d_head=128, d_mlp=18944,
                rope_theta=1000000.0)
C4_BASE = dict(vocab_size=152064, d_model=5120, n_heads=40, n_kv_heads=8, d_head=128, d_mlp=27648,
               rope_theta=1000000.0)
C4_DRAFT = dict(vocab_size=152064, d_model=896, n_heads=14, n_kv_heads=2, d_head=64, d_mlp=4864,
                rope_theta=1000000.0)

PAIRS = {"c2": (C2_BASE, C2_DRAFT), "c3": (C3_BASE, C3_DRAFT), "c4": (C4_BASE, C4_DRAFT)}

# trees as parent lists (-1 = child of the context tail); row 0 is the frontier
TREES = {
    1: [-1],
    6: [-1, 0, 1, 2, 3, 4],                                   # gamma = 5 chain verify
    9: [-1, 0, 0, 1, 1, 2, 2, 3, 5],                          # [2, 2, 1]-style verify tree
    16: [-1, 0, 0, 0, 1, 1, 2, 2, 3, 3, 4, 5, 6, 7, 8, 9],    # [3, 2, 1] verify tree
}
TREE37 = [-1] + [0] * 4 + [1 + i // 4 for i in range(16)] + [5 + i for i in range(16)]  # [4, 4, 1]


def _cfgs(pair, base_layers=2, draft_layers=4):
    b, d = PAIRS[pair]
    common = dict(max_positions=CTX + 64, weight_dtype=E.BF16, kv_dtype=E.BF16, tied_head=False)
    base = E.ModelConfig(n_layers=base_layers, seed=7, **b, **common)
    draft = E.ModelConfig(n_layers=draft_layers, seed=9, **d, **common)
    return base, draft


def _engine(pair):
    base, draft = _cfgs(pair)
    eng = E.Engine(base, draft, E.RunConfig(n=5, lp_size=2))
    eng.init_weights(E.Engine.BASE, base.seed, parity=False)
    eng.init_weights(E.Engine.DRAFT, draft.seed, parity=False)
    return eng, base, draft


def _torch_weights(eng, which, cfg):
    """The engine's bf16 weights (read back exactly, as fp32) -> fp64 on the GPU."""
    import torch
    d, H, Hkv, dh, f, V = cfg.d_model, cfg.n_heads, cfg.n_kv_heads, cfg.d_head, cfg.d_mlp, cfg.vocab_size
    dev = torch.device("cuda")
    W = {}

    def put(key, name, rows, cols, layer=-1):
        W[key] = torch.from_numpy(eng.read_tensor(which, name, rows, cols, layer=layer)).to(dev).double()

    put("embedding", "embedding", V, d)
    put("head", "head", d, V)
    put("final_norm_gain", "final_norm_gain", 1, d)
    W["final_norm_gain"] = W["final_norm_gain"][0]
    for l in range(cfg.n_layers):
        for name, shape in (("wq", (d, H * dh)), ("wk", (d, Hkv * dh)), ("wv", (d, Hkv * dh)),
                            ("wo", (H * dh, d)), ("w_gate", (d, f)), ("w_up", (d, f)), ("w_down", (f, d))):
            put(f"{name}.{l}", name, *shape, layer=l)
        for name in ("attn_norm_gain", "mlp_norm_gain"):
            put(f"{name}.{l}", name, 1, d, layer=l)
            W[f"{name}.{l}"] = W[f"{name}.{l}"][0]
    return W


def _plan_groups(spec):
    return [[int(x) for x in range(int(g.split("-")[0]), int(g.split("-")[-1]) + 1)] for g in spec.split("|")]


def _reference(W, cfg, prompt, trees, plan=None, bf16_acts=False, pos_shift=0):
    """fp64 logits / hidden of every tree row: the prompt as one precise chain
    pass (prefill), then all trees in ONE pass over the cached prompt (fuzzy
    under `plan`; disjoint ancestries: each tree row sees the prompt and its
    own ancestors only)."""
    import torch
    from tests import torch_ref
    parents, tokens, spans = [], [], []
    for toks, par in trees:
        off = len(parents)
        parents += [p if p < 0 else p + off for p in par]
        tokens += toks
        spans.append((off, off + len(par)))
    P = len(prompt)
    pos, mask = torch_ref.tree_rows(P, parents)
    pos[P:] += pos_shift  # negative control: a rotary off-by-one on the pass rows
    ns = SimpleNamespace(**cfg.__dict__)
    kv = {}
    with torch.no_grad():
        torch_ref.forward_rows(W, ns, prompt, pos[:P], mask[:P, :P], head_rows=torch.tensor([P - 1]).cuda(),
                               kv_out=kv, bf16_acts=bf16_acts)
        logits, h = torch_ref.forward_rows(W, ns, tokens, pos[P:], mask[P:, :],
                                           plan=_plan_groups(plan) if plan else None, past=kv, bf16_acts=bf16_acts)
    lg = logits.cpu().numpy()
    hid = h.cpu().numpy()
    return [(lg[a:b], hid[a:b]) for a, b in spans]


def _errs(got_l, got_h, ref_l, ref_h):
    """Per row: max |err| / RMS(ref) and ||err||_2 / ||ref||_2 of logits and hidden."""
    out = []
    for r in range(ref_l.shape[0]):
        dl, dh = got_l[r] - ref_l[r], got_h[r] - ref_h[r]
        out.append((np.abs(dl).max() / np.sqrt(np.mean(ref_l[r] ** 2)), np.linalg.norm(dl) / np.linalg.norm(ref_l[r]),
                    np.abs(dh).max() / np.sqrt(np.mean(ref_h[r] ** 2)), np.linalg.norm(dh) / np.linalg.norm(ref_h[r])))
    return np.array(out)


def _check(got_l, got_h, ref_l, ref_h, what, bound_max, bound_l2):
    e = _errs(got_l, got_h, ref_l, ref_h)
    print(f"{what}: logits max {e[:, 0].max():.2e} l2 {e[:, 1].max():.2e} | hidden max {e[:, 2].max():.2e} "
          f"l2 {e[:, 3].max():.2e}")
    assert e[:, [0, 2]].max() <= bound_max and e[:, [1, 3]].max() <= bound_l2, what
    for r in range(ref_l.shape[0]):
        rms_l = np.sqrt(np.mean(ref_l[r] ** 2))
        top2 = np.sort(ref_l[r])[-2:]
        if top2[1] - top2[0] > 2 * bound_max * rms_l:
            assert int(np.argmax(got_l[r])) == int(np.argmax(ref_l[r])), f"{what} row {r}: argmax differs"


@pytest.mark.parametrize("pair", ["c2", "c3", "c4"])
def test_bf16_kernels_at_baseline_shapes_vs_fp64(pair):
    import torch
    eng, base, draft = _engine(pair)
    rng = np.random.default_rng({"c2": 1, "c3": 2, "c4": 3}[pair])
    prompt = [int(t) for t in rng.integers(0, base.vocab_size, CTX)]
    for which, cfg, plan in ((E.Engine.BASE, base, None), (E.Engine.DRAFT, draft, "0|1-2|3")):
        trees, got = [], []
        for T, par in TREES.items():
            toks = [int(t) for t in rng.integers(0, cfg.vocab_size, T)]
            lg, h = eng.forward_tree(which, prompt, toks, par, plan=plan)
            trees.append((toks, par))
            got.append((lg, h))
        W = _torch_weights(eng, which, cfg)
        exact = _reference(W, cfg, prompt, trees, plan)
        shifted = _reference(W, cfg, prompt, trees[-1:], plan, pos_shift=1)
        del W
        torch.cuda.empty_cache()
        for (T, _), (gl, gh), (rl, rh) in zip(TREES.items(), got, exact):
            _check(gl, gh, rl, rh, f"{pair} {'base' if which else 'draft'} T={T}", BOUND_MAX, BOUND_L2)
        # the bound discriminates: a rotary off-by-one reference is far outside it
        e = _errs(got[-1][0], got[-1][1], shifted[0][0], shifted[0][1])
        assert e[:, 1].max() > 5 * BOUND_L2, e[:, 1].max()
    eng.close()


_POOL_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1]); sys.path.insert(0, sys.argv[1] + "/tests")
from test_gpu_bf16_shapes import _engine, TREE37, CTX
from paper_2502_02493_b200 import espec as E
eng, base, draft = _engine("c4")
rng = np.random.default_rng(11)
prompt = [int(t) for t in rng.integers(0, base.vocab_size, CTX)]
out = []
for which, cfg in ((E.Engine.BASE, base), (E.Engine.DRAFT, draft)):
    toks = [int(t) for t in rng.integers(0, cfg.vocab_size, len(TREE37))]
    lg, h = eng.forward_tree(which, prompt, toks, TREE37)
    out += [lg, h]
np.savez(sys.argv[2], *out)
"""


def test_decode_gemv_tail_pool_bitwise_above_16_rows(tmp_path):
    """> 16-row passes run as several 16-row launches that
    must not share tail-pool counters. A 37-row [4,4,1] verify pass on the C4
    shapes (small kcb, many problems for the 0.5B drafter) is bitwise equal
    with the tail pool on (default) and off (ESPEC_SG_POOL=0)."""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = []
    for pool in ("12", "0"):
        f = tmp_path / f"pool{pool}.npz"
        env = dict(os.environ, ESPEC_SG_POOL=pool)
        r = subprocess.run([sys.executable, "-c", _POOL_SCRIPT, root, str(f)], env=env, capture_output=True,
                           text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        z = np.load(f)
        res.append([z[k] for k in sorted(z.files, key=lambda s: int(s.split("_")[1]))])
    for other in res[1:]:
        for a, b in zip(res[0], other):
            assert np.array_equal(a, b)


@pytest.mark.parametrize("ppi", ["4", "8"])
def test_attention_cluster_combine_bitwise_equals_combine_kernel(tmp_path, ppi):
    """The split-context attention combines its chunks either inside a thread
    block cluster (DSMEM, default for 2..16 chunks) or through the workspace
    and the combine kernel (ESPEC_ATTN_CLUSTER=0). Both run one arithmetic
    (attn_tc.cu tca_combine), so a 37-row verify pass at ctx 2100 is bitwise
    equal either way: ppi 4 -> 9 chunks (a non-portable cluster), ppi 8 -> 5.
    The ticket combine (ESPEC_ATTN_COMBINE=ticket: the last chunk CTA to
    finish combines from the workspace) must match as well."""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = []
    for cl, comb in (("16", ""), ("0", ""), ("0", "ticket")):
        f = tmp_path / f"cl{cl}{comb}.npz"
        env = dict(os.environ, ESPEC_ATTN_CLUSTER=cl, ESPEC_ATTN_PPI=ppi, ESPEC_ATTN_COMBINE=comb)
        r = subprocess.run([sys.executable, "-c", _POOL_SCRIPT, root, str(f)], env=env, capture_output=True,
                           text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        z = np.load(f)
        res.append([z[k] for k in sorted(z.files, key=lambda s: int(s.split("_")[1]))])
    for other in res[1:]:
        for a, b in zip(res[0], other):
            assert np.array_equal(a, b)
