"""Summarise a CTA-pair forward timeline (tools/timeline.py output) of the even CTA.

MMA issuer (role 0): ev0 loop start j, ev1 S(j+1) issued, ev2 P(j) complete (both CTAs),
ev3 P V(j) issued.  Softmax warp 0 (role 1): ev0 S(j) seen, ev2 S loaded, ev3 slow path
taken, ev1 P(j) arrived."""
import sys

import numpy as np

t = np.load(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/timeline_fwd.npy").astype(np.int64)
base = t[t > 0].min()
t = np.where(t > 0, t - base, -1)
n = int((t[0, :, 0] >= 0).sum())
s = slice(4, n - 1)


def med(x):
    return float(np.median(x[s]))


m, x = t[0, :n], t[1, :n]
print("kv tiles", n, "period", float(np.diff(m[4:n, 0]).mean()))
print("MMA: start->S(j+1) issued", med(m[:, 1] - m[:, 0]), " ->P(j) ready", med(m[:, 2] - m[:, 1]),
      " ->PV(j) issued", med(m[:, 3] - m[:, 2]), " ->next start", med(np.r_[m[1:, 0] - m[:-1, 3], 0]))
print("softmax: phase", med(x[:, 1] - x[:, 0]), "(ld", med(x[:, 2] - x[:, 0]), "exp", med(x[:, 1] - x[:, 2]),
      ") wait next S", med(np.r_[x[1:, 0] - x[:-1, 1], 0]), " slow tiles", int((x[:, 3] >= 0).sum()))
print("P arrive (warp 0, even CTA) -> MMA sees all P", med(m[:, 2] - x[:, 1]))
print("S(j+1) issued -> softmax sees S(j+1)", med(np.r_[x[1:, 0] - m[:-1, 1], 0]))
