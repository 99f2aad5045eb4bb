"""decode_plane on the cfg2 R4 stream (k = 0, B = 4): the indexed plane
kernel for ncu (`-k regex:k_plane_indexed4`)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_1805_06019_b200 as rl  # noqa: E402

data, _ = bench.make_stream(bench.CFG)
st = rl.init(data)
for c in range(3):
    rl.decode_plane(st, 3, 4, c)
torch.cuda.synchronize()
