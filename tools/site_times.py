"""In-stream per-launch device time of each base-model kernel site (CUDA events
around the launch on the engine stream) in EasySpec verify (T = n+1) and
vanilla (T = 1) passes, C2 shapes."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import bench  # noqa: E402
from paper_2502_02493_b200 import espec as E  # noqa: E402

wl = bench.WORKLOADS["c2"]
mp = 512 + 200
base = E.ModelConfig(max_positions=mp, seed=7, tied_head=False, weight_dtype=E.BF16, kv_dtype=E.BF16, **wl["base"])
draft = E.ModelConfig(max_positions=mp, seed=9, tied_head=False, weight_dtype=E.BF16, kv_dtype=E.BF16, **wl["draft"])
# ESPEC_TP_PROXY=N: rank 0 of a TP-N group alone on this GPU (collectives loop back)
tp = int(os.environ.get("ESPEC_TP_PROXY", "1"))
eng = E.Engine(base, draft, E.RunConfig(algorithm="easyspec", n=5, lp_size=4, max_new_tokens=100), tp_size=tp)
if tp > 1:
    eng.link_loopback()
eng.init_weights(E.Engine.BASE, 7, parity=False)
eng.init_weights(E.Engine.DRAFT, 9, parity=False)
prompt = [int(t) for t in np.random.default_rng(1234).integers(0, base.vocab_size, size=512)]
names = {0: "qkv", 1: "attention", 2: "o", 3: "gate_up", 4: "down", 5: "head"}
for alg in ("easyspec", "vanilla"):
    for which, wname in ((1, "base"), (0, "draft")):
        if alg == "vanilla" and which == 0:
            continue
        row = []
        for kind in range(6):
            eng.set_run(E.RunConfig(algorithm=alg, n=5, lp_size=4, max_new_tokens=100))
            eng.begin(prompt)
            for _ in range(3):
                eng.step()
            eng.time_site(which, kind)
            for _ in range(4):
                eng.step()
            n, ms, by = eng.site_stats()
            eng.time_site(-1, -1)
            row.append(f"{names[kind]} {1e3 * ms / max(n, 1):6.1f}us x{n // 4}/step ({by / max(ms / max(n, 1), 1e-9) / 1e6 / 6543:.0%})")
        print(f"{alg:8s} {wname:5s} " + " | ".join(row), flush=True)
eng.close()
