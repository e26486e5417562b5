"""Summarise BSVD_CHASE_TRACE of the carried-block chase (k_chase2; development aid)."""
import sys
import numpy as np
t = np.fromfile(sys.argv[1], dtype=np.uint64).reshape(256, 32, 16).astype(np.int64)
ok = (t[:, :, 0] > 0) & (t[:, :, 7] > 0) & (t[:, :, 2] > 0) & (t[:, :, 4] > 0)
ok[:, 0] = False
names = ["dep wait", "msg wait", "new apply", "send", "carrier apply", "store+fence", "ordered rel"]
d = np.diff(t[:, :, :8], axis=2)
for i, nm in enumerate(names):
    v = d[:, :, i][ok]
    print(f"{nm:14s} median {np.median(v)/1e3:7.2f} us  mean {v.mean()/1e3:7.2f} us")
v = (t[:, :, 8] - t[:, :, 2])[ok]
print("loads done after msg: median %.2f us (negative: before)" % (np.median(v) / 1e3))
v = (t[:, :, 9] - np.maximum(t[:, :, 8], t[:, :, 2]))[ok]
print("reflector: median %.2f us" % (np.median(v) / 1e3))
v = (t[:, :, 3] - t[:, :, 9])[ok]
print("apply (dots+emit+update): median %.2f us" % (np.median(v) / 1e3))
# chain link: send(k+1) - send(k) within a sweep (steady part)
link = (t[:, 2:31, 4] - t[:, 1:30, 4])
lk = link[(t[:, 2:31, 4] > 0) & (t[:, 1:30, 4] > 0)]
print("chain link (send k -> send k+1) median %.2f us mean %.2f" % (np.median(lk) / 1e3, lk.mean() / 1e3))
# time from message sent (op k's pivot) to receiver start of apply: t2(k) - t4(k-1)
lat = t[:, 2:31, 2] - t[:, 1:30, 4]
lv = lat[(t[:, 2:31, 2] > 0) & (t[:, 1:30, 4] > 0)]
print("msg latency (sent -> received) median %.2f us" % (np.median(lv) / 1e3))
st = t[:, 0, 3]
st = st[st > 0]
print("sweep interval (op0 done) median %.2f us" % (np.median(np.diff(st)) / 1e3))
# dependency satisfied vs msg: which one gates the apply?
gate_dep = (t[:, 1:, 1] > t[:, 1:, 2])[ok[:, 1:]]
print("fraction of ops where dependency came after the message: %.2f" % gate_dep.mean())
