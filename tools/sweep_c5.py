"""BASELINE.json configs[4] (C5): layer-parallel width 1/2/4/8 x gamma 3-8 x
context 512-8K on the Llama-3-70B/8B shapes, one B200, greedy, bf16 random init.

Per point: EasySpec ms per iteration (calibrate / fuzzy draft / verify split)
and draft-stage ms per drafted token, beside vanilla and sequential-draft SD on
the same kernels. alpha ~ 0 for independent random-init models, so an
iteration emits one token; the draft-stage latency vs lp is the comparison the
paper's Fig. 4 makes (one GPU here: layer parallelism = batched group launches).

usage: python tools/sweep_c5.py [ctx,...] > gpurun_out/c5_sweep.jsonl
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2502_02493_b200 import espec as E  # noqa: E402

CTXS = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [512, 2048, 8192]
# ESPEC_C5_LPS / ESPEC_C5_NS override the grid (e.g. ESPEC_C5_NS=8,12,15 for 9-16 row verify passes)
LPS = [int(x) for x in os.environ.get("ESPEC_C5_LPS", "1,2,4,8").split(",")]
NS = [int(x) for x in os.environ.get("ESPEC_C5_NS", "3,5,8").split(",")]
WARM, STEPS = 2, 4


def main():
    wl = bench.WORKLOADS["c2"]
    mp = max(CTXS) + (WARM + STEPS + 2) * (max(NS) + 1) + 64
    base = E.ModelConfig(max_positions=mp, seed=7, tied_head=False, weight_dtype=E.BF16, kv_dtype=E.BF16, **wl["base"])
    draft = E.ModelConfig(max_positions=mp, seed=9, tied_head=False, weight_dtype=E.BF16, kv_dtype=E.BF16,
                          **wl["draft"])
    eng = E.Engine(base, draft, E.RunConfig(algorithm="easyspec", n=5, lp_size=4, max_new_tokens=64))
    eng.init_weights(E.Engine.BASE, 7, parity=False)
    eng.init_weights(E.Engine.DRAFT, 9, parity=False)
    stream = torch.cuda.ExternalStream(eng.stream())

    def run(alg, n, lp, prompt):
        eng.set_run(E.RunConfig(algorithm=alg, n=n, lp_size=lp, temperature=0.0,
                                max_new_tokens=(WARM + STEPS + 2) * (n + 1)))
        eng.begin(prompt)
        for _ in range(WARM):
            eng.step()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        trs, em = [], 0
        for _ in range(STEPS):
            out, tr = eng.step()
            em += len(out)
            trs.append(tr)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / STEPS
        return dict(alg=alg, n=n, lp=lp, ms_per_iter=ms, tokens_per_s=em / (STEPS * ms / 1e3),
                    calibrate_ms=sum(t.calibrate_ms for t in trs) / STEPS,
                    draft_ms=sum(t.draft_ms for t in trs) / STEPS,
                    verify_ms=sum(t.verify_ms for t in trs) / STEPS,
                    alpha=sum(t.m for t in trs) / max(1, sum(t.n for t in trs)))

    for ctx in CTXS:
        prompt = [int(t) for t in np.random.default_rng(1234).integers(0, base.vocab_size, size=ctx)]
        rows = [run("vanilla", 1, 1, prompt)]
        for n in NS:
            rows.append(run("sd", n, 1, prompt))
            for lp in LPS:
                rows.append(run("easyspec", n, lp, prompt))
        for r in rows:
            r["ctx"] = ctx
            # draft-stage ms per drafted token: (calibrate + fuzzy draft) / n
            r["draft_ms_per_drafted_token"] = (r["calibrate_ms"] + r["draft_ms"]) / r["n"] if r["alg"] != "vanilla" else 0
            print(json.dumps(r), flush=True)
    eng.close()


if __name__ == "__main__":
    main()
