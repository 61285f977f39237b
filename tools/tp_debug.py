import json, sys, os
sys.path.insert(0, os.getcwd())
from dataclasses import replace
from paper_2502_02493_b200 import espec as E
GEN = json.load(open("tests/golden/ref_generate.json"))
case = GEN[3]; r = case["run"]
base = E.ModelConfig(**{k: case["base"][k] for k in ("vocab_size","d_model","n_layers","n_heads","d_head","d_mlp","max_positions","norm_eps","seed")})
print(base, case["keep"], r, flush=True)
run = E.RunConfig(algorithm="vanilla", n=r["n"], widths=r["widths"], lp_size=r["lp_size"], temperature=0.0, max_new_tokens=8, seed=1)
engines = E.tp_group_local(base, replace(base, n_layers=case["keep"]), run, 2, truncated=case["keep"])
print("vanilla", E.tp_generate(engines, prompt=b"abc")[0][0], flush=True)
for e in engines: e.set_run(replace(run, algorithm="sd"))
print("sd", E.tp_generate(engines, prompt=b"abc")[0][0], flush=True)
