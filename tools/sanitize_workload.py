"""Small workload for compute-sanitizer (tools/gpu_sanitize.sh): the bf16
perf path end to end — tcgen05 prefill (tc_gemm_kernel), stream-K decode GEMV
(sgemv_kernel, 8- and 16-row variants, > 16-row two-pass launches, tail pool,
split-K tickets), tensor-core attention (attn_mma_kernel, tree mask), greedy
and T > 0 acceptance kernels — plus a TP-2 group's one-shot collectives
(allreduce / allgather kernels) with both shards on this GPU."""
import os
import sys
from dataclasses import replace

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from paper_2502_02493_b200 import espec as E  # noqa: E402

what = sys.argv[1] if len(sys.argv) > 1 else "all"
base = E.ModelConfig(vocab_size=4096, d_model=512, n_layers=4, n_heads=8, n_kv_heads=2, d_head=64, d_mlp=1536,
                     max_positions=512, seed=5, rope_theta=500000.0, tied_head=False, weight_dtype=E.BF16,
                     kv_dtype=E.BF16)
draft = replace(base, n_layers=4, seed=105)
prompt = [int(t) for t in np.random.default_rng(3).integers(0, 4096, 80)]
if what in ("all", "single"):
    for alg, widths, temp in (("easyspec", [1] * 5, 0.0), ("easyspec", [3, 2, 1, 1, 1], 0.0),
                              ("easyspec", [2, 2, 1, 1, 1], 0.8)):
        e = E.Engine(base, draft, E.RunConfig(algorithm=alg, n=5, widths=widths, lp_size=2, temperature=temp,
                                              max_new_tokens=12, seed=1))
        e.init_weights(E.Engine.BASE, base.seed, parity=False)
        e.init_weights(E.Engine.DRAFT, draft.seed, parity=False)
        toks, _ = e.generate_tokens(prompt)
        print(alg, widths, temp, toks, flush=True)
        # a 37-row [4,4,1] tree pass (two 16-row launches + one 5-row launch)
        par = [-1] + [0] * 4 + [1 + i // 4 for i in range(16)] + [5 + i for i in range(16)]
        lg, _ = e.forward_tree(E.Engine.BASE, prompt, list(range(37)), par)
        print("tree37 argmax", lg.argmax(-1)[:8], flush=True)
        e.close()
if what in ("all", "tp"):
    run = E.RunConfig(algorithm="easyspec", n=5, lp_size=2, temperature=0.0, max_new_tokens=12, seed=1)
    engines = E.tp_group_local(base, draft, run, 2, parity=False)
    res = E.tp_generate(engines, tokens=prompt)
    assert res[0][0] == res[1][0]
    print("tp2", res[0][0], flush=True)
    for e in engines:
        e.close()
print("workload done", flush=True)
