"""Per-phase cycle breakdown of the fused decode (debug build with
-DRLFC_PHASE_TIMING; first 4096 CTAs, per warp).

    python tools/phase_timing.py            # builds the debug .so if needed
"""
import ctypes
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1805_06019_b200 import _build, _native  # noqa: E402

DBG = os.path.join(ROOT, "paper_1805_06019_b200", "librlfc_b200_phase.so")
if not os.path.exists(DBG):
    cus = [os.path.join(_build.CSRC, f) for f in sorted(os.listdir(_build.CSRC)) if f.endswith(".cu")]
    subprocess.run(["/usr/local/cuda/bin/nvcc"] + _build.NVCC_FLAGS + ["-DRLFC_PHASE_TIMING", "-o", DBG] + cus,
                   check=True)
L = _native.load_library(DBG)
L.rlfc_debug_phase.argtypes = [ctypes.c_void_p]
_native._lib = L

import torch  # noqa: E402
import bench  # noqa: E402
import paper_1805_06019_b200 as rl  # noqa: E402
from paper_1805_06019_b200 import decoder  # noqa: E402

data, _ = bench.make_stream(bench.CFG)
st = rl.init(data)
hdr = st.header
out = torch.empty((hdr.s_count, hdr.t_count, hdr.height, hdr.width, 3), dtype=torch.uint8, device="cuda")
for _ in range(3):
    decoder.decode_field(st, 0, out=out)
torch.cuda.synchronize()
buf = np.zeros(4096 * 8 * 8, dtype=np.int64)
assert L.rlfc_debug_phase(buf.ctypes.data) == 0
ph = buf.reshape(4096, 8, 8)[:, :4]          # 4 warps per CTA
names = ["store+walk", "decode", "cls_masks", "barA", "items+prefill", "barB1", "blend", "barB2"]
tot = ph.sum(axis=2).mean()
print(f"cycles per CTA (mean over warps/CTAs): {tot:.0f}")
for w in range(4):
    row = ph[:, w].mean(axis=0)
    print(f"warp {w}: " + "  ".join(f"{n}={v:.0f}" for n, v in zip(names, row)))
