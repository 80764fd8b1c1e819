"""Summarise a forward timeline (tools/timeline.py output) of one CTA: medians per key tile.

MMA issuer (role 0): ev0 loop start j, ev1 P V_0(j-1) issued, ev2 S_0(j) issued, ev3 P V_1(j-1)
issued, ev4 S_1(j) issued.  Softmax warpgroup t (role 1 + t, warp 0 lane 0): ev0 S_t(j) seen,
ev2 S loaded, ev3 slow path taken (row max needed), ev1 P_t(j) arrived."""
import sys

import numpy as np

t = np.load(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/timeline_fwd.npy").astype(np.int64)
base = t[t > 0].min()
t = np.where(t > 0, t - base, -1)
n = int((t[0, :, 0] >= 0).sum())
s = slice(10, n - 1)


def med(x):
    return float(np.median(x[s]))


m = t[0, :n]
print("kv tiles", n, "period", float(np.diff(m[10:n, 0]).mean()))
print("MMA: start->PV0 issued", med(m[:, 1] - m[:, 0]), "->S0 issued", med(m[:, 2] - m[:, 1]), "->PV1 issued",
      med(m[:, 3] - m[:, 2]), "->S1 issued", med(m[:, 4] - m[:, 3]), "-> next start", med(np.r_[m[1:, 0] - m[:-1, 4], 0]))
for r in (1, 2):
    x = t[r, :n]
    print("softmax WG", r - 1, "phase", med(x[:, 1] - x[:, 0]), "(ld", med(x[:, 2] - x[:, 0]), "exp + P store",
          med(x[:, 1] - x[:, 2]), ") wait next S", med(np.r_[x[1:, 0] - x[:-1, 1], 0]),
          "slow-path tiles", int((x[:, 3] >= 0).sum()))
    # S_t(j) issued (MMA stamp) -> softmax sees S; P_t(j) arrived -> P V_t(j) issued in the next loop
    print("   S issue -> seen", med(x[:, 0] - m[:, 2 * r]), " P arrive -> PV issued(next j)",
          med(np.r_[m[1:, 2 * r - 1] - x[:-1, 1], 0]))
