"""Summarise a decode-megakernel timeline (ESPEC_MK_TRACE): per op, the
critical-path window [first consumer start .. last arrival], the spread of
consumer starts (dependency-wait skew), staging time and epilogue tail."""
import sys
import numpy as np

NAMES = {0: "embed", 1: "gemv", 2: "attn", 3: "add"}
EPI = {0: "store", 1: "resid", 2: "silu", 3: "qkv", 4: "argmax"}


def main(path, limit=40):
    ops = []
    for line in open(path):
        v = line.split()
        typ, epi, units = int(v[0]), int(v[1]), int(v[2])
        t = np.array([int(x) for x in v[3:]], dtype=np.int64).reshape(-1, 8)
        ops.append((typ, epi, units, t))
    t0 = min(o[3][:, 0].min() for o in ops)
    prev_end = t0
    rows = []
    for k, (typ, epi, units, t) in enumerate(ops):
        start_min, start_max = t[:, 0].min(), t[:, 0].max()
        staged = np.median(t[:, 1] - t[:, 0]) if typ == 1 else 0
        done_max = t[:, 2].max()
        arr_max = t[:, 3].max()
        name = NAMES[typ] + ("." + EPI[epi] if typ == 1 else "")
        rows.append((k, name, units, (start_min - prev_end) / 1e3, (start_max - start_min) / 1e3, staged / 1e3,
                     (done_max - start_min) / 1e3, (arr_max - done_max) / 1e3, (arr_max - prev_end) / 1e3))
        prev_end = arr_max
    total = (prev_end - t0) / 1e3
    print(f"total {total:.1f} us over {len(ops)} ops")
    print(f"{'k':>4} {'op':12s} {'units':>6} {'gap':>7} {'skew':>7} {'stage':>7} {'work':>8} {'tail':>7} {'span':>8}")
    agg = {}
    for r in rows:
        a = agg.setdefault(r[1], np.zeros(6))
        a += np.array([1, r[3], r[4], r[6], r[7], r[8]])
    for r in rows[:limit]:
        print(f"{r[0]:4d} {r[1]:12s} {r[2]:6d} {r[3]:7.2f} {r[4]:7.2f} {r[5]:7.2f} {r[6]:8.2f} {r[7]:7.2f} {r[8]:8.2f}")
    # attention internals (CTAs that ran an item): K loaded, V loaded, ticket, combine end
    att = [o[3] for o in ops if o[0] == 2]
    if att:
        ks, vs, tk, ce = [], [], [], []
        for t in att:
            m = t[:, 4] > 0
            ks += list((t[m, 4] - t[m, 0]) / 1e3)
            vs += list((t[m, 5] - t[m, 4]) / 1e3)
            mt = m & (t[:, 6] > 0)
            tk += list((t[mt, 6] - t[mt, 5]) / 1e3)
            me = t[:, 7] > 0
            ce += list((t[me, 7] - t[me, 6]) / 1e3)
        print(f"attention internals (median us): K {np.median(ks):.2f}  QK {np.median(vs):.2f}  "
              f"softmax {np.median(tk) if tk else 0:.2f}  Vwait {np.median(ce) if ce else 0:.2f}  "
              f"(max start->K {np.max(ks):.2f})")
    print("per op type (mean us): n gap skew work tail span")
    for k, a in agg.items():
        print(f"  {k:12s} n={int(a[0]):4d} gap={a[1]/a[0]:6.2f} skew={a[2]/a[0]:6.2f} work={a[3]/a[0]:8.2f} "
              f"tail={a[4]/a[0]:6.2f} span={a[5]/a[0]:8.2f} total={a[5]:9.1f}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
