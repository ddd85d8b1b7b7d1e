"""Analyse a ZOLO_TRACE dump of one DAG-scheduled forward sweep (sparse path).

Each task line: start_ns deps_done_ns done_ns (smid<<48 | chunk<<47 | i<<16 | ndeps),
in claim order. Prints the sweep span, busy fraction of
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
smid = (raw[:, 3] >> np.uint64(48)).astype(np.int64)
chunk = ((raw[:, 3] >> np.uint64(47)) & np.uint64(1)).astype(np.int64)
row = ((raw[:, 3] >> np.uint64(16)) & np.uint64(0x7FFFFFFF)).astype(np.int64)
nd = (raw[:, 3] & np.uint64(0xFFFF)).astype(np.int64)
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

# the last block rows to complete (the sweep's tail chain): row-task completion times
rt = chunk == 0
last = {}
for k in np.where(rt)[0]:
    last[row[k]] = max(last.get(row[k], 0.0), done[k])
rows_by_done = sorted(last.items(), key=lambda kv: kv[1])
tail = rows_by_done[-40:]
print("last 40 block rows to finish (row: done us, gap to previous):")
prev = None
line = []
for r_, t_ in tail:
    line.append(f"{r_}:{t_:.0f}(+{(t_ - prev) if prev is not None else 0:.1f})")
    prev = t_
print("  " + " ".join(line))

# CTA-time breakdown (needs the 6-word trace: wait ns and first-tile-ready stamps)
if raw.shape[1] >= 6:
    wait_ns = raw[:, 4].astype(np.float64) / 1e3
    first = (raw[:, 5].astype(np.float64) - t0) / 1e3
    has_first = raw[:, 5] > 0
    startup = np.where(has_first, first - claim, ready - claim)
    loop = np.where(has_first, ready - first, 0.0)
    tail_t = done - ready
    ncta = 296
    tot = ncta * span
    print(f"CTA-time breakdown over {ncta} CTAs x span: startup (claim..first tile) {startup.sum() / tot:.1%}, "
          f"tile loop {np.maximum(loop - wait_ns, 0).sum() / tot:.1%}, dependency waits {wait_ns.sum() / tot:.1%}, "
          f"epilogue {tail_t.sum() / tot:.1%}, idle/claim gaps {1 - (done - claim).sum() / tot:.1%}")
    print(f"per task us: startup median {np.median(startup):.2f}, epilogue median {np.median(tail_t):.2f}, "
          f"waits mean {wait_ns.mean():.2f}")
    tiles = nd + (1 - chunk)  # + pre entry (upper bound)
    busy = np.maximum(loop - wait_ns, 1e-3)
    m = tiles >= 4
    print(f"tile-loop rate (tasks with >= 4 entries): median {np.median(busy[m] / tiles[m]):.2f} us per tile per CTA")
