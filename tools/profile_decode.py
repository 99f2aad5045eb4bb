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
ap.add_argument("--preset", default="R4", help="cfg2 bitrate preset (tools/bitrate_sweep.py)")
a = ap.parse_args()
cfg = bench.CFG
if a.preset != "R4":
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    from bitrate_sweep import PRESETS
    h, B, s, tp, tb = PRESETS[a.preset]
    cfg = dict(bench.CFG, h=h, B=B, shift=s, tp=tp, tb=tb)
data, _ = bench.make_stream(cfg)
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
