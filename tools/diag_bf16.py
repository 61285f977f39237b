"""Diagnostic: where does the bf16 path's error vs fp64 come from? Runs
espec_forward_tree on small variants (1 layer, short / long prompt) and prints
error vs the exact and the bf16-rounding-emulating fp64 reference."""
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from dataclasses import replace
import numpy as np
import torch
from paper_2502_02493_b200 import espec as E
import test_gpu_bf16_shapes as S

pair = sys.argv[1] if len(sys.argv) > 1 else "c4"
for L in (2, 4):
    base, draft = S._cfgs(pair, base_layers=L, draft_layers=2)
    eng = E.Engine(base, draft, E.RunConfig(n=5, lp_size=1))
    eng.init_weights(E.Engine.BASE, base.seed, parity=False)
    eng.init_weights(E.Engine.DRAFT, draft.seed, parity=False)
    W = S._torch_weights(eng, E.Engine.BASE, base)
    rng = np.random.default_rng(5)
    for P in (1, 4, 16, 17, 300, 2100):
        prompt = [int(t) for t in rng.integers(0, base.vocab_size, P)]
        toks = [int(rng.integers(0, base.vocab_size))]
        lg, h = eng.forward_tree(E.Engine.BASE, prompt, toks, [-1])
        for emu in (False, True):
            (rl, rh), = S._reference(W, base, prompt, [(toks, [-1])], None, bf16_acts=emu)
            e = S._errs(lg, h, rl, rh)[0]
            print(f"{pair} L={L} P={P} {'emul ' if emu else 'exact'}: logits max {e[0]:.2e} l2 {e[1]:.2e} | hidden max {e[2]:.2e} l2 {e[3]:.2e}", flush=True)
    del W
    eng.close()
    torch.cuda.empty_cache()
