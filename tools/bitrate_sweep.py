"""cfg2 bitrate ladder (presets R1-R6): full-field
decode throughput of the staged and fused paths per preset, with achieved
bpp, present fraction and the roofline fraction by algorithmic bytes.

    python tools/bitrate_sweep.py [--out profiles/r2_bitrate_sweep.json]

Streams come from the native producer (byte-identical to the reference
encoder) and are cached under data/.  Each preset's staged and fused outputs
are checked bit-exact against the per-block kernel before timing (CUDA
events, 10 timed decodes after 3 warm-ups; the 0.9 GB output exceeds L2).
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_1805_06019_b200 as rl  # noqa: E402
from paper_1805_06019_b200 import decoder  # noqa: E402

PRESETS = {   # h, B, s, Tp, Tb
    "R1": (5, 16, 6, 64, 1_000_000),
    "R2": (4, 8, 5, 32, 6_000),
    "R3": (3, 4, 5, 24, 2_000),
    "R4": (3, 4, 4, 16, 1_000),
    "R5": (3, 4, 4, 16, 500),
    "R6": (3, 4, 3, 8, 300),
}


def time_decode(st, out, kernel, iters=10):
    for _ in range(3):
        decoder.decode_field(st, 0, out=out, kernel=kernel, check=False)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        decoder.decode_field(st, 0, out=out, kernel=kernel, check=False)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r2_bitrate_sweep.json"))
    ap.add_argument("--presets", default="R1,R2,R3,R4,R5,R6")
    a = ap.parse_args()
    peak, peak_kind = bench.peaks()
    rows = []
    for name in a.presets.split(","):
        h, B, s, tp, tb = PRESETS[name]
        cfg = dict(bench.CFG, h=h, B=B, shift=s, tp=tp, tb=tb)
        data, _ = bench.make_stream(cfg)
        st = rl.init(data)
        hdr = st.header
        stats = bench.stream_stats(st)
        out = torch.empty((hdr.s_count, hdr.t_count, hdr.height, hdr.width, 3),
                          dtype=torch.uint8, device="cuda")
        ref, _ = decoder.decode_field(st, 0, kernel="simple")
        row = {"preset": name, "h": h, "B": B, "shift": s, "Tp": tp, "Tb": tb,
               "stream_bytes": len(data), "bpp": round(stats["bpp"], 4),
               "present_frac": round(stats["present_frac"], 5)}
        alg = stats["comp_bytes"] + stats["root_bytes"] + stats["out_bytes"]
        npix = hdr.s_count * hdr.t_count * hdr.width * hdr.height
        for kernel in ("staged", "fused"):
            got, _ = decoder.decode_field(st, 0, kernel=kernel)
            exact = bool(torch.equal(got, ref))
            ms = time_decode(st, out, kernel)
            row[kernel] = {"ms": round(ms, 4), "gpix_per_s": round(npix / ms / 1e6, 1),
                           "hbm_frac": round(alg / (ms * 1e-3) / 1e9 / peak, 4),
                           "exact_vs_per_block_kernel": exact}
        row["alg_bytes"] = int(alg)
        rows.append(row)
        print(json.dumps(row), flush=True)
        del out, ref, st
        torch.cuda.empty_cache()
    res = {"workload": "cfg2 17x17x1024^2 seed 7, PNG roots, full-field decode",
           "peak_gbs": peak, "peak_source": peak_kind, "rows": rows}
    with open(a.out, "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
