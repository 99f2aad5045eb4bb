"""Minimal driver for ncu captures of the decode kernels (one GPU).

    python tools/profile_decode.py [--kernel staged|fused|simple] [--iters N]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_1805_06019_b200 as rl  # noqa: E402
from paper_1805_06019_b200 import decoder  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--kernel", default="staged")
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--render", type=int, default=0)
a = ap.parse_args()
data, _ = bench.make_stream(bench.CFG)
st = rl.init(data)
hdr = st.header
out = torch.empty((hdr.s_count, hdr.t_count, hdr.height, hdr.width, 3),
                  dtype=torch.uint8, device="cuda")
for _ in range(a.iters):
    decoder.decode_field(st, 0, out=out, kernel=a.kernel)
if a.render:
    poses = [rl.SlabPose(1.5 + 0.05 * i, 3.25 + 0.03 * i, 512, 512)
             for i in range(a.render)]
    rl.render_views(st, poses)
torch.cuda.synchronize()
print("ok")
