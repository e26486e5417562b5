"""Summarise BSVD_CHASE_TRACE phase timestamps (development aid)."""
import os, sys
import numpy as np
t = np.fromfile(sys.argv[1], dtype=np.uint64).reshape(256, 32, 8).astype(np.int64)
ok = (t[:, :, 0] > 0) & (t[:, :, 5] > 0)
names = ["poll", "gen", "csync1", "slice", "fence+csync2+rel"]
d = np.stack([t[:, :, 1] - t[:, :, 0], t[:, :, 2] - t[:, :, 1], t[:, :, 3] - t[:, :, 2],
              t[:, :, 4] - t[:, :, 3], t[:, :, 5] - t[:, :, 4]], -1)
sel = d[ok]
print("ops traced", sel.shape[0])
for k, nm in enumerate(names):
    print(f"{nm:18s} median {np.median(sel[:, k])/1e3:7.2f} us  mean {sel[:, k].mean()/1e3:7.2f} us")
# sweep start interval
st = t[:, 0, 1]
st = st[st > 0]
print("sweep start interval median", np.median(np.diff(st)) / 1e3, "us")
