import sys, os
sys.path.insert(0, "/root/repo")
import numpy as np
from dataclasses import replace
from paper_2502_02493_b200 import espec as E
base = E.ModelConfig(vocab_size=4096, d_model=512, n_layers=2, n_heads=8, n_kv_heads=2, d_head=64, d_mlp=1536,
                     max_positions=512, seed=5, rope_theta=500000.0, tied_head=False, weight_dtype=E.BF16, kv_dtype=E.BF16)
e = E.Engine(base, replace(base, seed=6), E.RunConfig(n=3, lp_size=1))
e.init_weights(E.Engine.BASE, 5, parity=False); e.init_weights(E.Engine.DRAFT, 6, parity=False)
lg, h = e.forward(E.Engine.BASE, [1, 2, 3])
print("done", lg.argmax(-1))
