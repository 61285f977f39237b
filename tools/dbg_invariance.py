import sys, numpy as np
sys.path.insert(0, '.')
from dataclasses import replace
from paper_2502_02493_b200 import espec as E
base = E.ModelConfig(vocab_size=4096, d_model=512, n_layers=6, n_heads=8, n_kv_heads=2, d_head=64, d_mlp=1536,
                     max_positions=1024, seed=5, rope_theta=500000.0, tied_head=False, weight_dtype=E.BF16, kv_dtype=E.BF16)
draft = replace(base, n_layers=4, seed=105)
eng = E.Engine(base, draft, E.RunConfig(n=5, lp_size=2))
eng.init_weights(E.Engine.BASE, 5, parity=False); eng.init_weights(E.Engine.DRAFT, 105, parity=False)
toks = [int(t) for t in np.random.default_rng(17).integers(0, 4096, size=16)]
res = {}
for T in (1, 8, 9, 16):
    lg, h = eng.forward(E.Engine.BASE, toks[:T])
    kv = [eng.cache_view(E.Engine.BASE, l, 0, 1) for l in range(6)]
    res[T] = (lg[0], h[0], kv)
for T in (8, 9, 16):
    print("T", T, "logits eq", np.array_equal(res[1][0], res[T][0]), "hidden eq", np.array_equal(res[1][1], res[T][1]),
          "max|dh|", float(np.abs(res[1][1] - res[T][1]).max()),
          "kv eq per layer", [bool(np.array_equal(res[1][2][l][0], res[T][2][l][0]) and np.array_equal(res[1][2][l][1], res[T][2][l][1])) for l in range(6)])
