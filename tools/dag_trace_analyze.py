"""Analyse a ZOLO_TRACE dump of one DAG-scheduled forward sweep (sparse path).

Each task line: claim_ns deps_ready_ns done_ns (smid<<32 | ndeps); tasks are
ordered (block row s, chain, group). Prints the sweep span, busy fraction of
the resident CTAs over time (10 bins), the tail after 90% of tasks finished,
and per-task duration vs dependency count.
"""
import sys

import numpy as np

path = sys.argv[1]
hdr = open(path).readline().split()
raw = np.loadtxt(path, dtype=np.uint64, comments="#")
raw = raw[raw[:, 0] > 0]
claim, ready, done = (raw[:, k].astype(np.float64) for k in range(3))
smid = (raw[:, 3] >> np.uint64(32)).astype(np.int64)
nd = (raw[:, 3] & np.uint64(0xFFFFFFFF)).astype(np.int64)
t0 = claim.min()
claim, ready, done = (claim - t0) / 1e3, (ready - t0) / 1e3, (done - t0) / 1e3
span = done.max()
dur = done - claim
wait = ready - claim
print(" ".join(hdr[1:]))
print(f"tasks {len(raw)}  span {span:.1f} us  SMs used {len(np.unique(smid))}")
print(f"task us: mean {dur.mean():.2f} median {np.median(dur):.2f}  dep-wait median {np.median(wait):.2f} "
      f"mean {wait.mean():.2f}  compute median {np.median(done - ready):.2f}")
busy = dur.sum()
ncta = len(np.unique(smid)) * max(1, round(len(raw) / max(1, len(np.unique(smid))) / 1e9))
print(f"sum task time / span = {busy / span:.1f} concurrent tasks on average")
bins = np.linspace(0, span, 11)
for a, b in zip(bins[:-1], bins[1:]):
    ov = np.clip(np.minimum(done, b) - np.maximum(claim, a), 0, None).sum() / (b - a)
    ovc = np.clip(np.minimum(done, b) - np.maximum(ready, a), 0, None).sum() / (b - a)
    print(f"  [{a:8.1f},{b:8.1f}) us  active {ov:6.1f}  computing {ovc:6.1f}")
order = np.sort(done)
t90 = order[int(0.9 * len(order))]
print(f"90% of tasks done at {t90:.1f} us; tail {span - t90:.1f} us ({100 * (span - t90) / span:.0f}% of span)")
for lo, hi in ((0, 4), (4, 16), (16, 64), (64, 256), (256, 1 << 30)):
    m = (nd >= lo) & (nd < hi)
    if m.any():
        print(f"  deps [{lo},{hi}): {m.sum():6d} tasks, compute median {np.median(done[m] - ready[m]):7.2f} us "
              f"({np.median((done[m] - ready[m]) / np.maximum(nd[m], 1)):.3f} us/dep), wait median {np.median(wait[m]):.2f}")
