"""BASELINE.json configs[0] (C1): the reference CLI's default pair — base
init_model(12 layers, d 64, 4 heads x 16, d_mlp 128, vocab 258, seed 7) and
its first-8-layer truncated drafter, greedy, n = 4, widths 1, lp 2, prompt
"the quick brown fox", 256 new tokens — end to end on both sides:

  reference: oracle/_ref/ref_bench c1 (the unmodified reference core, 1 core)
  ours:      espec_generate through the C ABI on cuda:0, fp32 parity mode
             (weights bit-identical to init_model), tokens checked against
             the oracle restatement of the same run.
"""
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_2502_02493_b200 import espec as E  # noqa: E402

PROMPT = b"the quick brown fox"
NEW = 256


def ours(alg):
    base = E.ModelConfig(vocab_size=258, d_model=64, n_layers=12, n_heads=4, d_head=16, d_mlp=128,
                         max_positions=512, seed=7)
    run = E.RunConfig(algorithm=alg, n=4, widths=[1, 1, 1, 1], lp_size=2, temperature=0.0, max_new_tokens=NEW)
    eng = E.truncated_pair(base, 8, run)
    eng.generate(PROMPT)  # warm-up
    best, toks = 1e30, None
    for _ in range(5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        toks, traces = eng.generate(PROMPT)
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    eng.close()
    ob = O.Model(O.ModelConfig(vocab_size=258, d_model=64, n_layers=12, n_heads=4, d_head=16, d_mlp=128,
                               max_positions=512, norm_eps=1e-5, seed=7))
    ref = O.generate(ob, ob.truncated(8), O.RunConfig(algorithm=alg, n=4, lp_size=2, temperature=0.0,
                                                       max_new_tokens=NEW, seed=1), PROMPT, with_cache=False)
    return len(toks) / best, best, toks == ref.tokens, ref.alpha


def reference(alg):
    exe = os.path.join(ROOT, "oracle", "_ref", "ref_bench")
    out = subprocess.run([exe, "c1", alg, str(NEW), "5"], capture_output=True, text=True, check=True).stdout
    return json.loads(out.strip().splitlines()[-1])


def main():
    print(f"C1, {NEW} new tokens, greedy; ours = one B200 through the C ABI (wall clock per generate call), "
          f"reference = oracle/_ref/ref_bench c1 (1 core, best of 5)")
    for alg in ("vanilla", "sd", "easyspec"):
        tps, s, same, alpha = ours(alg)
        r = reference(alg)
        print(f"{alg:9s} ours {tps:9.1f} tok/s ({s * 1e3:7.2f} ms)  reference {r['tokens_per_s']:9.1f} tok/s "
              f"({r['ms']:8.2f} ms)  speed-up {tps / r['tokens_per_s']:5.2f}x  tokens == oracle: {same}  "
              f"alpha {alpha:.3f}", flush=True)


if __name__ == "__main__":
    main()
