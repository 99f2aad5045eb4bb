"""Time the full-field decode of the bench workload under several launch
settings (environment knobs read at launch time) in one process.

    python tools/sweep_decode.py 'RLFC_BLEND_THREADS=128 RLFC_BLEND_TW=64' \
        'RLFC_BLEND_THREADS=256 RLFC_BLEND_TW=128' [--kernel staged]

Each argument is one setting: space-separated NAME=VALUE pairs.  Prints one
line per setting: Gpix/s and ms per decode (CUDA events, 20 timed calls
after 3 warm-up calls, output 0.9 GB > L2).
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
ap.add_argument("settings", nargs="*", default=[""])
ap.add_argument("--kernel", default="staged")
ap.add_argument("--iters", type=int, default=20)
a = ap.parse_args()
data, _ = bench.make_stream(bench.CFG)
st = rl.init(data)
hdr = st.header
out = torch.empty((hdr.s_count, hdr.t_count, hdr.height, hdr.width, 3),
                  dtype=torch.uint8, device="cuda")
ref, _ = decoder.decode_field(st, 0, kernel="simple")
npix = hdr.s_count * hdr.t_count * hdr.width * hdr.height
for setting in a.settings:
    pairs = [p.split("=", 1) for p in setting.split()]
    saved = {k: os.environ.get(k) for k, _ in pairs}
    for k, v in pairs:
        os.environ[k] = v
    for _ in range(3):
        decoder.decode_field(st, 0, out=out, kernel=a.kernel, check=False)
    torch.cuda.synchronize()
    ok = torch.equal(out, ref)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.iters):
        decoder.decode_field(st, 0, out=out, kernel=a.kernel, check=False)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.iters
    print(f"{setting or '(default)':50s} {npix / ms / 1e6:8.1f} Gpix/s "
          f"{ms:.4f} ms  exact={ok}", flush=True)
    for k, v in saved.items():
        if v is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = v
