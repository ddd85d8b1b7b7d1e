"""Analyse a ZOLO_TRACE dump (16 slots per block row, step order, ns):
owner [0] start [6] critical product done [1] saw c_i [7] stores+barrier [2] published x_i;
helper [3] start [10] pipeline start [8] far tiles done [9] #far tiles [4] all tiles done [5] published c_i."""
import sys

import numpy as np

raw = np.loadtxt(sys.argv[1], dtype=np.float64)
nfar = raw[:, 9].copy()
t = raw.copy()
t[:, 9] = 0
t0 = t[t > 0].min()
t = np.where(t > 0, t - t0, np.nan) / 1e3  # us
c = lambda k: t[:, k]
med = np.nanmedian
step = np.diff(c(2))
print(f"steps {len(t)}, total {c(2)[-1] - c(2)[0]:.1f} us, per step mean {np.nanmean(step):.2f} median {med(step):.2f}")
print(f"owner : start->product {med(c(6) - c(0)):.2f} | ->saw c {med(c(1) - c(6)):.2f} | ->stored+bar {med(c(7) - c(1)):.2f} | ->published {med(c(2) - c(7)):.2f}")
print(f"helper: start->pipeline {med(c(10) - c(3)):.2f} | far tiles {med(c(8) - c(10)):.2f} us for {np.median(nfar):.0f} tiles "
      f"({med((c(8) - c(10)) / np.maximum(nfar, 1)):.2f} us/tile) | near {med(c(4) - c(8)):.2f} | ->published {med(c(5) - c(4)):.2f}")
print(f"far tiles done -> x_(i-3) published (slack, +: waits): {med(c(2)[:-3] - c(8)[3:]):.2f} us")
print(f"x_(i-2) published -> helper all tiles done {med(c(4)[2:] - c(2)[:-2]):.2f} | -> c published {med(c(5)[2:] - c(2)[:-2]):.2f}")
print(f"helper c_i published -> owner saw c_i {med(c(1) - c(5)):.2f} us")
if raw.shape[1] > 12 and (raw[:, 11] > 0).any():
    print(f"owner detail: start->barrier1 {med(c(11) - c(0)):.2f} | barrier1->product done {med(c(12) - c(11)):.2f} | "
          f"->after release {med(c(6) - c(12)):.2f}")
