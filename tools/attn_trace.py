"""Summarise an attention timeline (ESPEC_ATTN_TRACE=n): per CTA the times of
start, dependency release, first K page, pages done, partial written and (the
last CTA of each kv head / m-tile) combine done, in us relative to the earliest
CTA start."""
import sys

import numpy as np

lines = open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/attn_trace.txt").read().split("\n")
print(lines[0])
t = np.array([[int(x) for x in l.split()] for l in lines[1:] if l.strip()], dtype=np.int64)
t0 = t[t[:, 0] > 0, 0].min()
names = ["cta start", "dep released", "first K page", "pages done", "partial written", "combine done",
         "cluster synced", "rank0 combined"]
for e, n in sorted(enumerate(names), key=lambda x: [0, 1, 2, 3, 4, 6, 7, 5][x[0]]):
    v = t[:, e]
    v = (v[v > 0] - t0) / 1e3
    if len(v):
        print(f"  {n:18s} n {len(v):4d} min {v.min():8.2f}  median {np.median(v):8.2f}  max {v.max():8.2f} us")
