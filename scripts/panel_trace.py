"""Summarise BSVD_PANEL_TRACE (development aid)."""
import sys
import numpy as np
t = np.fromfile(sys.argv[1], dtype=np.uint64)[:9 * 64 * 8].reshape(9 * 64, 8).astype(np.int64)
names = ["load", "qr", "Rsave+G", "T", "V/U write"]
leaf = t[:64]
ok = leaf[:, 5] > 0
d = np.diff(leaf[ok][:, :6], axis=1)
print("leaves", ok.sum(), " ".join(f"{n}={np.median(d[:, i])/1e3:.1f}us" for i, n in enumerate(names)),
      " total", np.median(leaf[ok][:, 5] - leaf[ok][:, 0]) / 1e3, "us")
t0 = leaf[ok][:, 0].min()
for j in range(1, 8):
    tt = t[64 + j * 64: 64 + (j + 1) * 64]
    ok = tt[:, 5] > 0
    if not ok.any():
        continue
    d = np.diff(tt[ok][:, :6], axis=1)
    print(f"level {j}: nodes {ok.sum()} " + " ".join(f"{n}={np.median(d[:, i])/1e3:.1f}us" for i, n in enumerate(names)),
          f" start@{(tt[ok][:, 0].min() - t0)/1e3:.1f}us end@{(tt[ok][:, 5].max() - t0)/1e3:.1f}us")
if t.size >= 0:
    raw = np.fromfile(sys.argv[1], dtype=np.uint64).astype(np.int64)
    if raw.size >= 64 * 9 * 8 + 256:
        st = raw[64 * 9 * 8: 64 * 9 * 8 + 128]
        ph = raw[64 * 9 * 8 + 128: 64 * 9 * 8 + 256]
        base = raw[1]  # leaf 0 mark(1)
        if st[0] > 0:
            d = np.diff(np.r_[base, st])
            print("leaf0 column-step us:", np.round(d[:8] / 1e3, 2), "... median", np.median(d) / 1e3)
            print("leaf0 phase stamps (us from start):", np.round((ph[:16][ph[:16] > 0] - base) / 1e3, 1))
