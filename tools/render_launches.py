"""Launch list of small-batch slab renders (cfg2 R4 stream, 512^2): warm-up,
then batch 1 at k = 0 and k = h and batch 64 at k = 0, each bracketed by a
marker kernel so the ncu launch list splits by call.

    ncu --metrics gpu__time_duration.sum --clock-control none --csv \\
        --log-file gpurun_out/render_launches.csv python tools/render_launches.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_1805_06019_b200 as rl  # noqa: E402

data, _ = bench.make_stream(bench.CFG)
st = rl.init(data)
h = st.header.tree_height
rng = np.random.default_rng(5)
one = [rl.SlabPose(7.3, 4.6, 512, 512)]
many = [rl.SlabPose(float(rng.uniform(0, 16)), float(rng.uniform(0, 16)), 512, 512) for _ in range(64)]
mark = torch.zeros(1, device="cuda")
for _ in range(3):
    rl.render_views(st, one)
    rl.render_views(st, one, stop_level=h)
    rl.render_views(st, many)
torch.cuda.synchronize()
for name, poses, k in (("b1k0", one, 0), ("b1kh", one, h), ("b64k0", many, 0)):
    mark.add_(1)                         # marker: elementwise kernel
    rl.render_views(st, poses, stop_level=k)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    for _ in range(20):
        rl.render_views(st, poses, stop_level=k)
    ev[1].record()
    torch.cuda.synchronize()
    print(name, round(ev[0].elapsed_time(ev[1]) / 20, 4), "ms")
mark.add_(1)
torch.cuda.synchronize()
