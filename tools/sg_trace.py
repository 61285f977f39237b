"""Summarise decode-GEMV timelines (ESPEC_SG_TRACE="K,N,T,n[,cnt]"): per
launch, per CTA the times of start, dependency release, staging done, consumers done, epilogues done — in us relative to the earliest
CTA start of the FIRST traced launch, so gaps between consecutive launches
show up directly."""
import sys

import numpy as np

lines = open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/sg_trace.txt").read().split("\n")
heads = [l for l in lines if l.startswith("epi")]
rows = [l for l in lines if l.strip() and not l.startswith("epi")]
t = np.array([[int(x) for x in l.split()] for l in rows], dtype=np.int64).reshape(len(heads), -1, 16)
t0 = t[0][t[0][:, 0] > 0, 0].min()
names = {0: "cta start", 1: "dep released", 5: "x rows landed", 6: "x batch stored", 2: "staged", 3: "consumers done",
         4: "epilogues done"}
for h, tl in zip(heads, t):
    print(h)
    for e in (0, 1, 5, 6, 2, 3, 4):
        v = tl[:, e]
        v = (v[v > 0] - t0) / 1e3
        if len(v):
            print(f"  {names[e]:20s} min {v.min():8.2f}  median {np.median(v):8.2f}  max {v.max():8.2f} us")
