"""Summarise a fused-step evict-item timeline (EPK_STEP_TRACE dump)."""
import sys
import numpy as np

path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/step_trace.bin"
raw = open(path, "rb").read()
C, L, nsm, _ = np.frombuffer(raw[:16], np.uint32)
h = np.frombuffer(raw[16:], np.uint64)
n = int(h[0])
rec = h[8:8 + 4 * n].reshape(n, 4)
score_end = h[8 + 4 * 60000: 8 + 4 * 60000 + nsm].astype(np.int64)
start = h[8 + 4 * 60000 + 512: 8 + 4 * 60000 + 512 + nsm].astype(np.int64)
t0 = start.min()
item = (rec[:, 0] & 0xffffffff).astype(np.int64)
layer = (rec[:, 0] >> 32).astype(np.int64)
ts, te = rec[:, 2].astype(np.int64) - t0, rec[:, 3].astype(np.int64) - t0
print(f"C={C} L={L} items={n} kernel span {(max(te.max(), (score_end - t0).max())) / 1e3:.1f} us, scoring end "
      f"min/med/max {(score_end - t0).min() / 1e3:.1f}/{np.median(score_end - t0) / 1e3:.1f}/{(score_end - t0).max() / 1e3:.1f} us")
# classify by r within layer using the decode order is complex: infer from durations per layer
order = np.argsort(ts)
for l in range(int(L)):
    m = layer == l
    if not m.any():
        continue
    print(f"layer {l:2d}: items {m.sum():4d} first start {ts[m].min() / 1e3:8.1f} last end {te[m].max() / 1e3:8.1f} "
          f"busy sum {(te[m] - ts[m]).sum() / 1e3:8.1f} us")


def classify(j, C, L):
    if j == 0:
        return 0
    jp = j - 1
    t, q = 1 + jp // (C + 1), jp % (C + 1)
    return 0 if (t <= L - 1 and q == 0) else 1


names = ["prep", "gather"]
kind = np.array([classify(int(j), int(C), int(L)) for j in item])
dur = (te - ts) / 1e3
wait = (rec[:, 1] >> 16).astype(np.int64) / 1e3
for k, nm in enumerate(names):
    m = kind == k
    if m.any():
        print(f"{nm:8s} n={m.sum():5d} dur us: median {np.median(dur[m]):7.1f} p90 {np.percentile(dur[m], 90):7.1f} "
              f"max {dur[m].max():7.1f} sum {dur[m].sum():9.1f}  wait median {np.median(wait[m]):7.1f} sum {wait[m].sum():9.1f}")
# gather items after scoring ended
se = np.median(score_end - t0)
m = (kind == 1) & (ts > se)
if m.any():
    print(f"gather items starting after scoring end: {m.sum()}, median dur {np.median(dur[m]):.1f} us")

px = h[8 + 4 * 60000 + 2048: 8 + 4 * 60000 + 2048 + 4 * int(L)].reshape(int(L), 4).astype(np.int64) / 1e3
print("prep phases (us from item start): bin / cand scan / resolve / keep+counts")
for l in range(int(L)):
    print(l, px[l].round(1).tolist())
