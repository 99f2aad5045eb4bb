"""One 10^6-pick decode_blocks batch (cfg2 R4, k = 0) for ncu
(`-k regex:k_blocks_indexed`)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1805_06019_b200 as rl  # noqa: E402
from paper_1805_06019_b200 import decoder  # noqa: E402

data, _ = bench.make_stream(bench.CFG)
st = rl.init(data)
hdr = st.header
wb, hb = hdr.block_grid
rng = np.random.default_rng(7)
n = 1_000_000
req = np.stack([rng.integers(0, hdr.s_count, n), rng.integers(0, hdr.t_count, n), rng.integers(0, wb, n),
                rng.integers(0, hb, n), rng.integers(0, 3, n), np.zeros(n, np.int64)], 1).astype(np.int32)
dreq = torch.from_numpy(req).cuda()
for _ in range(3):
    decoder.decode_blocks(st, dreq, raise_errors=False)
torch.cuda.synchronize()
