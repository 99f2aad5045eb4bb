"""Where a batch-1 slab render's wall time goes (cfg2 R4 stream, 512^2):
wall time of render_views, of the native batch call alone, and a
torch.profiler trace of 20 calls (kernel and copy times from CUPTI, gaps
between them)."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_1805_06019_b200 as rl  # noqa: E402
from paper_1805_06019_b200 import renderer  # noqa: E402

data, _ = bench.make_stream(bench.CFG)
st = rl.init(data)
h = st.header.tree_height
one = [rl.SlabPose(7.3, 4.6, 512, 512)]
for _ in range(20):
    rl.render_views(st, one)
    rl.render_views(st, one, stop_level=h)
torch.cuda.synchronize()
res = {}
for name, k in (("b1k0", 0), ("b1kh", h)):
    t0 = time.perf_counter()
    for _ in range(200):
        rl.render_views(st, one, stop_level=k)
    torch.cuda.synchronize()
    res[name + "_render_views_us"] = (time.perf_counter() - t0) / 200 * 1e6
    # the native call alone (Python argument preparation hoisted)
    captured = {}
    real = renderer._render_slab_batch

    def grab(*a, **kw):
        captured["a"] = a
        return real(*a, **kw)
    renderer._render_slab_batch = grab
    rl.render_views(st, one, stop_level=k)
    renderer._render_slab_batch = real
    a = captured["a"]
    t0 = time.perf_counter()
    for _ in range(200):
        real(*a)
    torch.cuda.synchronize()
    res[name + "_render_slab_batch_us"] = (time.perf_counter() - t0) / 200 * 1e6
print(json.dumps(res))
from torch.profiler import ProfilerActivity, profile  # noqa: E402
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    for _ in range(20):
        rl.render_views(st, one)
    torch.cuda.synchronize()
os.makedirs("gpurun_out", exist_ok=True)
prof.export_chrome_trace("gpurun_out/render_trace.json")
print(prof.key_averages().table(sort_by="self_cuda_time_total", row_limit=20))
