"""Read a forward timeline (tools/timeline.py) of the round-2 block forward: per key tile j,
MMA stamps (0 before S(j), 1 after S(j) issued, 2 after PV(j-1) issued), softmax warpgroup
stamps (0 S(j) seen, 2 row max exchanged, 1 P(j) arrived), TMA stamp 0 (K(j) issued)."""
import sys

import numpy as np

t = np.load(sys.argv[1] if len(sys.argv) > 1 else 'gpurun_out/timeline_fwd.npy').astype(np.int64)
base = t[t > 0].min()
t = np.where(t > 0, t - base, -1)
n = int((t[0, :, 0] >= 0).sum())
s = slice(8, n - 2)
med = lambda x: float(np.median(x[s]))  # noqa: E731
print('kv tiles', n, 'period', med(np.diff(t[0, :n, 0])))
print('MMA: S(j) issue', med(t[0, :n, 1] - t[0, :n, 0]), ' PV(j-1) wait+issue', med(t[0, :n, 2] - t[0, :n, 1]),
      ' -> next', med(np.r_[t[0, 1:n, 0] - t[0, :n - 1, 2], 0]))
for r in (1, 2):
    print(f'softmax WG {r - 1}: S seen->max xch', med(t[r, :n, 2] - t[r, :n, 0]), ' ->P arrive',
          med(t[r, :n, 1] - t[r, :n, 2]), ' P arrive->next S seen', med(np.r_[t[r, 1:n, 0] - t[r, :n - 1, 1], 0]))
    print('   S(j) issued -> seen', med(t[r, :n, 0] - t[0, :n, 1]), '  P(j) arrive -> PV(j) issued',
          med(t[0, 1:n, 2] - t[r, :n - 1, 1]))
print('TMA K(j) issue -> S(j) issue start', med(t[0, :n, 0] - t[3, :n, 0]))
# issuer detail (stamps 3: K(j) ready, 4: P(j) ready seen by the issuer, 5: V(j) ready)
print('issuer: start S(j) -> K(j) ready', med(t[0, :n, 3] - t[0, :n, 0]), ' K ready -> S issued', med(t[0, :n, 1] - t[0, :n, 3]))
print('issuer: S(j) issued -> P(j-1) seen', med(t[0, 1:n, 4][:n - 1] - t[0, 1:n, 1]) if False else
      med(np.r_[t[0, :n - 1, 4] - t[0, 1:n, 1], 0]), ' P seen -> V ready', med(t[0, :n, 5] - t[0, :n, 4]))
print('TMA: waiting for the K stage release', med(t[3, :n, 0] - t[3, :n, 1]))
