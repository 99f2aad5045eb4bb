"""Driver for ncu captures of the non-headline kernels (one GPU): the
batched slab render (render_views, 64 x 512^2 views from the cfg2 stream:
tap-camera decode + k_render_slab), a pinhole render, a 10^6-pick
random-access batch (k_blocks_indexed), single-block decodes
(k_decode_block_one) and the init-time PNG root unfilter (k_unfilter).

    python tools/profile_misc.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_1805_06019_b200 as rl  # noqa: E402
from paper_1805_06019_b200 import decoder  # noqa: E402

data, _ = bench.make_stream(bench.CFG)
st = rl.init(data)                       # k_unfilter (PNG roots)
hdr = st.header
rng = np.random.default_rng(11)
poses = [rl.SlabPose(float(rng.uniform(0, 16)), float(rng.uniform(0, 16)), 512, 512) for _ in range(64)]
for _ in range(2):
    rl.render_views(st, poses)
rl.render_view(st, rl.CameraPose(eye=(8.0, 8.0, -2.0), look=(0.0, 0.0, 1.0), fov_deg=50.0, width=512, height=512))
wb, hb = hdr.block_grid
n = 1_000_000
req = np.stack([rng.integers(0, 17, n), rng.integers(0, 17, n), rng.integers(0, wb, n), rng.integers(0, hb, n),
                rng.integers(0, 3, n), np.zeros(n, np.int64)], 1).astype(np.int32)
dreq = torch.from_numpy(req).cuda()
for _ in range(2):
    decoder.decode_blocks(st, dreq, raise_errors=False)
for p in req[:4]:
    rl.decode_block(st, (int(p[0]), int(p[1])), (int(p[2]), int(p[3])), int(p[4]))
torch.cuda.synchronize()
print("ok")
