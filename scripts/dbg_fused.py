import sys; sys.path.insert(0, '.')
import numpy as np, torch
import paper_2509_17396_b200 as gpu
from tests.test_gpu_step_fused import _build, _run_fused, _generic
rng = np.random.default_rng(1024 + 512 + 64 + 128)
L, Hq, H, p = 3, 24, 8, 128
counts = [[1280] * 8, [1000, 1500, 0, 77, 1280, 2000, 640, 129], [300] * 8]
M = [1024, 512, 64]
slack = 128
layers, qs, kps, cin, q, kp, cap = _build(gpu, rng, L, Hq, H, p, counts, slack, 0.0)
cout, scores, kept = _run_fused(gpu, cin, q, kp, M, slack, "max", cap, 2000)
cref = _generic(gpu, cin, scores, M, slack, cap)
for l in range(L):
    a = cout.retained_positions()[l]; b = cref.retained_positions()[l]
    for h in range(H):
        if a[h] != b[h]:
            A, B = np.array(a[h]), np.array(b[h])
            d = np.nonzero(A != B)[0]
            print("layer", l, "head", h, "len", len(A), len(B), "first diff at", d[:5], "A", A[d[0]-2:d[0]+6].tolist(), "B", B[d[0]-2:d[0]+6].tolist(),
                  "sets equal", set(A.tolist()) == set(B.tolist()))
            break
print("kept", kept.tolist())
