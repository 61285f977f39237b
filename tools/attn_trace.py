"""Summarise an attention timeline (ESPEC_ATTN_TRACE=T,n; slots in attn_tc.cu
kTcaTraceSlots): per CTA the times of start, dependency release, first K page,
pages done, end and cluster sync in us relative to the earliest CTA start, then
the per-step pipeline (median over CTAs, us from the CTA's first K page):
QK(s) issued, S(s) seen by softmax, P(s) written, PV(s) issued, PV(s) seen."""
import sys

import numpy as np

lines = open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/attn_trace.txt").read().split("\n")
print(lines[0])
t = np.array([[int(x) for x in l.split()] for l in lines[1:] if l.strip()], dtype=np.int64)
t0 = t[t[:, 0] > 0, 0].min()
names = {0: "cta start", 6: "prologue issued", 7: "K page 0 landed", 1: "dep released", 54: "Q rows stored (t0)", 55: "page ids read", 53: "Q tile written",
         2: "first QK issued", 3: "pages done", 5: "cluster synced", 56: "combine done", 57: "cluster synced 2", 4: "end"}
for e in (0, 6, 7, 1, 54, 55, 53, 2, 3, 5, 56, 57, 4):
    if e >= t.shape[1]:
        continue
    v = t[:, e]
    v = (v[v > 0] - t0) / 1e3
    if len(v):
        print(f"  {names[e]:18s} n {len(v):4d} min {v.min():8.2f}  median {np.median(v):8.2f}  max {v.max():8.2f} us")
if t.shape[1] >= 48:
    print("  step   QK issued   S seen  P written  PV issued  PV seen   (median us from first K page)")
    k0 = t[:, 2]
    for s in range(8):
        cols = [8 + s, 24 + s, 40 + s, 16 + s, 32 + s]
        ok = (t[:, cols] > 0).all(axis=1) & (k0 > 0)
        if not ok.any():
            break
        med = [np.median((t[ok, c] - k0[ok]) / 1e3) for c in cols]
        print(f"  {s:4d} " + " ".join(f"{x:9.2f}" for x in med))
if t.shape[1] >= 64:
    ok = (t[:, 26] > 0) & (t[:, 48] > 0)
    if ok.any():
        base = t[ok, 26]
        lab = ["scores loaded", "row max exchanged", "exp summed", "fold done", "P stored", "P arrived"]
        cols = [48, 49, 50, 51, 52, 42]
        print("  step 2 softmax phases (median us from S(2) seen): " +
              ", ".join(f"{n} {np.median((t[ok, c] - base) / 1e3):.2f}" for n, c in zip(lab, cols)))
