"""BASELINE.md section 3 on the GPU box's host: the LIVE reference (rlfc 0.1.0,
numba backend, installed into baseline/_ref by pip --target; not part of the
product, not used by bench.py) timed on the cfg2 R4 workload.

    NUMBA_CACHE_DIR=/tmp/numba_cache python tools/reference_cpu_baselines.py \\
        [--out profiles/r2_reference_cpu_baselines.json]

The stream is the bench stream (bench.make_stream: GPU-built, sha256-equal to
the reference encoder's).  Measured: decode_image single-thread (8 views),
decode_image over all 289 views on a fork Pool(nproc), decode_block mean over
10,000 picks from default_rng(7) (test_acceptance.py:169-177), and
render_view(SlabPose 512x512) single-thread and pooled over poses.
"""
import argparse
import json
import multiprocessing as mp
import os
import platform
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
sys.path.insert(1, ROOT)

import numpy as np  # noqa: E402

_st = None


def _init(data):
    global _st
    from rlfc import decoder
    _st = decoder.init(data)


def _img(i):
    from rlfc import decoder
    s, t = divmod(i, _st.header.t_count)
    return decoder.decode_image(_st, (s, t)).nbytes


def _render(p):
    from rlfc import renderer
    s, t = p
    return renderer.render_view(_st, renderer.SlabPose(s, t, 512, 512)).nbytes


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r2_reference_cpu_baselines.json"))
    a = ap.parse_args()
    import bench
    import numba
    import rlfc
    from rlfc import decoder, kernels, renderer
    assert os.path.dirname(rlfc.__file__).startswith(os.path.join(ROOT, "baseline", "_ref")), rlfc.__file__
    data, _ = bench.make_stream(bench.CFG)
    nproc = os.cpu_count()
    res = {"reference": "rlfc 0.1.0 from baseline/_ref (pip --target of /root/reference/pkg), numba backend "
                        f"= {kernels.USE_NUMBA}", "numba": numba.__version__, "numpy": np.__version__,
           "cpu": platform.processor() or platform.machine(), "nproc": nproc,
           "workload": "cfg2 R4 17x17x1024^2 (bench stream, 70,053,079 B)"}
    try:
        with open("/proc/cpuinfo") as f:
            res["cpu"] = next(ln.split(":", 1)[1].strip() for ln in f if ln.startswith("model name"))
    except (OSError, StopIteration):
        pass
    t0 = time.perf_counter()
    st = decoder.init(data)
    res["init_s"] = round(time.perf_counter() - t0, 3)
    hdr = st.header
    decoder.decode_block(st, (0, 0), (0, 0), 0)            # JIT warm-up
    decoder.decode_image(st, (0, 0))
    # single thread decode_image
    views = [(s, 8) for s in range(0, 16, 2)]
    t0 = time.perf_counter()
    for v in views:
        decoder.decode_image(st, v)
    dt = time.perf_counter() - t0
    px = hdr.width * hdr.height
    res["decode_image_1core"] = {"views": len(views), "s_per_view": round(dt / len(views), 4),
                                 "mpix_per_s": round(len(views) * px / dt / 1e6, 3)}
    print(json.dumps(res["decode_image_1core"]), flush=True)
    # all 289 views over a fork pool
    n = hdr.s_count * hdr.t_count
    with mp.get_context("fork").Pool(nproc, _init, (data,)) as pool:
        pool.map(_img, range(nproc))                        # warm every worker
        t0 = time.perf_counter()
        pool.map(_img, range(n), chunksize=1)
        dt = time.perf_counter() - t0
    res["decode_all_pool"] = {"procs": nproc, "s": round(dt, 3), "mpix_per_s": round(n * px / dt / 1e6, 3),
                              "gpix_per_s": round(n * px / dt / 1e9, 5)}
    print(json.dumps(res["decode_all_pool"]), flush=True)
    # decode_block latency
    rng = np.random.default_rng(7)
    wb, hb = hdr.block_grid
    picks = rng.integers(0, [hdr.s_count, hdr.t_count, wb, hb, 3], size=(10000, 5))
    t0 = time.perf_counter()
    for s, t, bx, by, c in picks:
        decoder.decode_block(st, (int(s), int(t)), (int(bx), int(by)), int(c))
    res["decode_block_us"] = round((time.perf_counter() - t0) / len(picks) * 1e6, 2)
    print("decode_block", res["decode_block_us"], "us", flush=True)
    # render_view 512x512 slab poses
    prng = np.random.default_rng(5)
    poses = [(float(prng.uniform(0, 16)), float(prng.uniform(0, 16))) for _ in range(2 * nproc)]
    renderer.render_view(st, renderer.SlabPose(poses[0][0], poses[0][1], 64, 64))
    t0 = time.perf_counter()
    for s, t in poses[:2]:
        renderer.render_view(st, renderer.SlabPose(s, t, 512, 512))
    dt = time.perf_counter() - t0
    res["render_view_1core"] = {"views": 2, "s_per_view": round(dt / 2, 3), "views_per_s": round(2 / dt, 4)}
    print(json.dumps(res["render_view_1core"]), flush=True)
    with mp.get_context("fork").Pool(nproc, _init, (data,)) as pool:
        t0 = time.perf_counter()
        pool.map(_render, poses, chunksize=1)
        dt = time.perf_counter() - t0
    res["render_view_pool"] = {"procs": nproc, "views": len(poses), "views_per_s": round(len(poses) / dt, 3)}
    print(json.dumps(res["render_view_pool"]), flush=True)
    with open(a.out, "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
