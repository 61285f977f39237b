"""tcgen05 prompt-prefill GEMM (tc_gemm.cu): UMMA M=128 x N=256 tiles with
TMEM accumulators, checked against numpy on the same bf16-rounded operands
(fp32 accumulation on both sides: tolerance 1e-3 relative to the output
scale), including ragged M (not a multiple of 128) and N (not a multiple of
256), plus an end-to-end bf16 prefill through the engine vs the decode path."""
import ctypes as C
from dataclasses import replace

import numpy as np
import pytest

from paper_2502_02493_b200 import espec as E

pytestmark = pytest.mark.gpu


def _bf16(a):
    u = np.ascontiguousarray(a, np.float32).view(np.uint32)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000).astype(np.uint32)
    return r.view(np.float32)


@pytest.mark.parametrize("M,K,N", [(128, 256, 256), (200, 512, 768), (40, 4096, 1056), (256, 1024, 512)])
def test_tc_gemm_matches_numpy(M, K, N):
    L = E.lib()
    L.espec_probe_tc.argtypes = [C.c_int] * 3 + [C.c_void_p] * 3 + [C.c_int]
    rng = np.random.default_rng(M + K + N)
    x = rng.standard_normal((M, K)).astype(np.float32)
    w = (rng.standard_normal((K, N)) * 0.05).astype(np.float32)
    out = np.zeros((M, N), np.float32)
    assert L.espec_probe_tc(M, K, N, x.ctypes.data, w.ctypes.data, out.ctypes.data, 0) == 0
    ref = _bf16(x).astype(np.float64) @ _bf16(w).astype(np.float64)
    scale = np.abs(ref).max()
    np.testing.assert_allclose(out, ref, atol=1e-3 * scale, rtol=1e-3)


def test_prefill_then_decode_greedy_lossless_long_prompt():
    """A 300-token prompt: its first 299 rows go through tcgen05 chunks for
    both vanilla and speculative decoding, the last prompt row through the
    decode GEMV in both, so greedy outputs stay identical."""
    base = E.ModelConfig(vocab_size=4096, d_model=512, n_layers=4, n_heads=8, n_kv_heads=2, d_head=64, d_mlp=1536,
                         max_positions=512, seed=5, rope_theta=500000.0, tied_head=False, weight_dtype=E.BF16,
                         kv_dtype=E.BF16)
    draft = replace(base, n_layers=3, seed=105)
    prompt = [int(t) for t in np.random.default_rng(0).integers(0, 4096, 300)]
    outs = {}
    for alg in ("vanilla", "easyspec"):
        eng = E.Engine(base, draft, E.RunConfig(algorithm=alg, n=4, lp_size=2, temperature=0.0, max_new_tokens=20))
        eng.init_weights(E.Engine.BASE, base.seed, parity=False)
        eng.init_weights(E.Engine.DRAFT, draft.seed, parity=False)
        outs[alg], _ = eng.generate_tokens(prompt)
        eng.close()
    assert outs["easyspec"] == outs["vanilla"]
