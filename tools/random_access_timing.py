"""Random-access batch throughput (decode_blocks, 10^6 picks, k = 0) on the
cfg2 R4 stream, CUDA events; checks the blocks against the per-block kernel."""
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
                rng.integers(0, hb, n), rng.integers(0, 3, n), rng.integers(0, hdr.tree_height + 1, n)],
               1).astype(np.int32)
for k0 in (True, False):
    r = req.copy()
    if k0:
        r[:, 5] = 0
    dreq = torch.from_numpy(r).cuda()
    for _ in range(3):
        out, status = decoder.decode_blocks(st, dreq, raise_errors=False)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        decoder.decode_blocks(st, dreq, raise_errors=False)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    sub = r[:4096]
    ref = np.stack([rl.decode_block_progressive(st, (int(a[0]), int(a[1])), (int(a[2]), int(a[3])), int(a[4]),
                                                int(a[5])) for a in sub])
    got = out[:4096].cpu().numpy().reshape(ref.shape)
    print(f"k={'0' if k0 else 'mixed'}: {ms:.4f} ms per 10^6 blocks, {n / ms / 1e6:.2f} G blocks/s, "
          f"first 4096 equal to decode_block: {np.array_equal(got, ref)}", flush=True)
