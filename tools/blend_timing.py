"""Per-phase wall-clock breakdown of k_blend tiles (debug build with
-DRLFC_BLEND_TIMING: %globaltimer stamps by thread 0 of the first 65,536
CTAs of the last decode).

    python tools/blend_timing.py [--preset R4]
"""
import argparse
import ctypes
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
from paper_1805_06019_b200 import _build, _native  # noqa: E402

DBG = os.path.join(ROOT, "paper_1805_06019_b200", "librlfc_b200_btime.so")
if not os.path.exists(DBG):
    cus = [os.path.join(_build.CSRC, f) for f in sorted(os.listdir(_build.CSRC)) if f.endswith(".cu")]
    subprocess.run(["/usr/local/cuda/bin/nvcc"] + _build.NVCC_FLAGS + ["-DRLFC_BLEND_TIMING", "-o", DBG] + cus,
                   check=True)
L = _native.load_library(DBG)
L.rlfc_debug_blend.argtypes = [ctypes.c_void_p]
_native._lib = L

import torch  # noqa: E402
import bench  # noqa: E402
import paper_1805_06019_b200 as rl  # noqa: E402
from paper_1805_06019_b200 import decoder  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--preset", default="R4")
a = ap.parse_args()
cfg = bench.CFG
if a.preset != "R4":
    from bitrate_sweep import PRESETS
    h, B, s, tp, tb = PRESETS[a.preset]
    cfg = dict(bench.CFG, h=h, B=B, shift=s, tp=tp, tb=tb)
data, _ = bench.make_stream(cfg)
st = rl.init(data)
hdr = st.header
out = torch.empty((hdr.s_count, hdr.t_count, hdr.height, hdr.width, 3), dtype=torch.uint8, device="cuda")
for _ in range(3):
    decoder.decode_field(st, 0, out=out)
torch.cuda.synchronize()
buf = np.zeros(65536 * 8, dtype=np.int64)
assert L.rlfc_debug_blend(buf.ctypes.data) == 0
t = buf.reshape(65536, 8).astype(np.float64)
ok = (t > 0).all(axis=1)
t = t[ok]
d = np.diff(t, axis=1)
names = ["records", "sync1", "units", "tma wait+sync2", "tasks", "sync3", "store+read"]
life = t[:, 7] - t[:, 0]
span = t[:, 7].max() - t[:, 0].min()
print(f"tiles sampled {len(t)}; blend span {span / 1e3:.1f} us; tile lifetime mean {life.mean() / 1e3:.2f} us "
      f"p50 {np.median(life) / 1e3:.2f} p90 {np.percentile(life, 90) / 1e3:.2f}")
for n, col in zip(names, d.T):
    print(f"  {n:16s} mean {col.mean() / 1e3:6.2f} us  p50 {np.median(col) / 1e3:6.2f}  p90 {np.percentile(col, 90) / 1e3:6.2f}")
starts = np.sort(t[:, 0])
print(f"  concurrent tiles (mean) {life.sum() / span:.0f}")
