"""Time the C2 prompt prefill (512-token prompt -> first token) end to end.

ESPEC_PROFILE_REGION=1: ncu --profile-from-start off captures one request."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2502_02493_b200 import espec as E  # noqa: E402

ctx = int(sys.argv[1]) if len(sys.argv) > 1 else 512
wl = bench.WORKLOADS["c2"]
mp = ctx + 256
base = E.ModelConfig(max_positions=mp, seed=7, tied_head=False, weight_dtype=E.BF16, kv_dtype=E.BF16, **wl["base"])
draft = E.ModelConfig(max_positions=mp, seed=9, tied_head=False, weight_dtype=E.BF16, kv_dtype=E.BF16, **wl["draft"])
eng = E.Engine(base, draft, E.RunConfig(algorithm="easyspec", n=5, lp_size=4, max_new_tokens=1))
eng.init_weights(E.Engine.BASE, 7, parity=False)
eng.init_weights(E.Engine.DRAFT, 9, parity=False)
prompt = [int(t) for t in np.random.default_rng(1234).integers(0, base.vocab_size, size=ctx)]
for _ in range(2):
    eng.generate_tokens(prompt)
torch.cuda.synchronize()
reps = 3
t0 = time.perf_counter()
for _ in range(reps):
    eng.generate_tokens(prompt)
torch.cuda.synchronize()
dt = (time.perf_counter() - t0) / reps
print(f"prefill+first token, ctx {ctx}: {dt * 1e3:.1f} ms per request")
if os.environ.get("ESPEC_PROFILE_REGION") == "1":
    torch.cuda.profiler.start()
    eng.generate_tokens(prompt)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
eng.close()
