"""Time daba_coarse_blocks (SURVEY NEXT-3 building block) on a config: CUDA events on the launching stream."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import paper_2305_07026_b200 as daba  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "final13682"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 10
p = gen.generate(cfg)
cams_native = np.zeros((p.M, 15))
aa = np.asarray(p.cams, np.float64).reshape(-1, 9)
# BAL -> native (R = Exp(aa)^T, t = -R t_w2c, d = (f, f k1, f k2)) with torch on the host (timing input only)
th = np.linalg.norm(aa[:, :3], axis=1, keepdims=True)
k = aa[:, :3] / np.maximum(th, 1e-300)
K = np.zeros((p.M, 3, 3))
K[:, 0, 1], K[:, 0, 2], K[:, 1, 2] = -k[:, 2], k[:, 1], -k[:, 0]
K = K - K.transpose(0, 2, 1)
Rw2c = np.eye(3) + np.sin(th)[:, :, None] * K + (1 - np.cos(th))[:, :, None] * (K @ K)
R = Rw2c.transpose(0, 2, 1)
cams_native[:, :9] = R.reshape(-1, 9)
cams_native[:, 9:12] = -np.einsum("mij,mj->mi", R, aa[:, 3:6])
cams_native[:, 12] = aa[:, 6]
cams_native[:, 13] = aa[:, 6] * aa[:, 7]
cams_native[:, 14] = aa[:, 6] * aa[:, 8]
order = np.argsort(p.obs_cam, kind="stable")
off = np.concatenate([[0], np.cumsum(np.bincount(p.obs_cam, minlength=p.M))]).astype(np.int64)
dev = torch.device("cuda:0")
t = lambda a, dt: torch.as_tensor(np.ascontiguousarray(a), dtype=dt).to(dev)  # noqa: E731
args = (t(cams_native, torch.float64), t(np.asarray(p.pts).reshape(-1, 3), torch.float64),
        t(np.asarray(p.obs_pt)[order], torch.int32), t(np.asarray(p.obs_uv).reshape(-1, 2)[order], torch.float64),
        t(off, torch.int64))
for _ in range(2):
    daba.coarse_blocks(*args, loss=p.loss)
torch.cuda.synchronize()
st = torch.cuda.current_stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
for _ in range(n):
    out = daba.coarse_blocks(*args, loss=p.loss)
e1.record(st)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / n  # includes the V/gl memsets and the mirror kernel (and the output allocations)
# algorithmic bytes: per observation u 16 + point index 4 + point gather 24 + W 216; per camera 120 read + 91 write;
# per point V / gl 12 doubles (read-modify-write of the atomics counted once each way)
byts = p.K * (16 + 4 + 24 + 216) + p.M * (120 + 91 * 8) + p.N * 12 * 8 * 2
print(json.dumps({"config": cfg, "K": p.K, "ms": ms, "GB_per_s": byts / ms / 1e6, "bytes": byts,
                  "F": float(out[5].sum().item())}))
