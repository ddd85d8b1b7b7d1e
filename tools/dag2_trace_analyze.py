"""Analyse a ZOLO_TRACE dump of one v2 (warp-specialised) DAG forward sweep.

Task words: [0] producer claim, [2] consumer epilogue done, [3] smid<<48 | chunk<<47 | i<<16 | tile
products, [4] producer dependency-wait ns, [5] producer finished issuing the task (all ns).
"""
import sys

import numpy as np

path = sys.argv[1]
print(open(path).readline().strip())
raw = np.loadtxt(path, dtype=np.uint64, comments="#")
raw = raw[(raw[:, 0] > 0) & (raw[:, 2] > 0)]
t0 = raw[:, 0].min()
claim = (raw[:, 0] - t0).astype(np.float64) / 1e3
done = (raw[:, 2] - t0).astype(np.float64) / 1e3
issued = (raw[:, 5] - t0).astype(np.float64) / 1e3
wait = raw[:, 4].astype(np.float64) / 1e3
info = raw[:, 3]
tiles = (info & np.uint64(0xFFFF)).astype(np.float64)
chunk = ((info >> np.uint64(47)) & np.uint64(1)).astype(int)
row = ((info >> np.uint64(16)) & np.uint64(0x7FFFFFFF)).astype(int)
span = done.max()
print(f"tasks {len(raw)}, span {span:.1f} us, tile products {tiles.sum():.0f} "
      f"-> {tiles.sum() / span:.1f} tiles/us (DMMA-peak bound ~142 tiles/us for unmasked tiles)")
print(f"producer dependency waits: total {wait.sum() / 1e3:.1f} ms over {len(np.unique(raw[:, 3] >> np.uint64(48)))} SMs "
      f"({wait.sum() / (296 * span):.1%} of producer time), tasks that waited {np.mean(wait > 0):.1%}")
print(f"task latency claim->done median {np.median(done - claim):.2f} us, issue span median {np.median(issued - claim):.2f} us")
bins = np.linspace(0, span, 21)
for a, b in zip(bins[:-1], bins[1:]):
    m = (done >= a) & (done < b)
    act = np.clip(np.minimum(done, b) - np.maximum(claim, a), 0, None).sum() / (b - a)
    print(f"  [{a:8.1f},{b:8.1f}) us  tiles/us {tiles[m].sum() / (b - a):6.1f}  tasks in flight {act:6.1f}  "
          f"producer wait {np.clip(wait[m], 0, None).sum() / (b - a):6.1f}")
order = np.sort(done)
t90 = order[int(0.9 * len(order))]
print(f"90% of tasks done at {t90:.1f} us; tail {span - t90:.1f} us ({100 * (span - t90) / span:.0f}% of span)")
