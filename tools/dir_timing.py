"""Per-tile phase timing of k_field_dir (debug build with -DRLFC_DIR_TIMING).

Builds a timing variant of the library into scratch/, decodes the cfg2 bench
stream through it (the DeviceField / directory come from the product
library; device memory is shared), and prints the median per-tile phase
durations of the first 16 CTAs.  Test/measurement infrastructure only.
"""
import ctypes
import glob
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def build_debug(out, extra=()):
    from paper_1805_06019_b200 import _build
    cus = [os.path.join(_build.CSRC, f) for f in sorted(os.listdir(_build.CSRC)) if f.endswith(".cu")]
    subprocess.run(["nvcc"] + _build.NVCC_FLAGS + ["-DRLFC_DIR_TIMING", *extra, "-o", out] + cus, check=True)


def main():
    import torch
    import paper_1805_06019_b200 as rl
    path = sys.argv[1] if len(sys.argv) > 1 and sys.argv[1] else glob.glob(os.path.join(ROOT, "data", "bench_*.rlfc"))[0]
    extra = sys.argv[2].split(",") if len(sys.argv) > 2 and sys.argv[2] else []
    so = os.path.join(ROOT, "scratch", "librlfc_dirtiming%s.so" % ("_".join(e.strip("-D") for e in extra)))
    build_debug(so, extra)
    D = ctypes.CDLL(so)
    st = rl.init(open(path, "rb").read())
    df = st.device_field()
    dr = df.directory()
    hdr = st.header
    out = torch.empty((hdr.s_count, hdr.t_count, hdr.height, hdr.width, 3), dtype=torch.uint8, device="cuda")
    status = torch.zeros(1, dtype=torch.int64, device="cuda")
    fn = D.rlfc_decode_field_dir
    fn.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                   ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    k = int(sys.argv[3]) if len(sys.argv) > 3 else 0
    for it in range(4):
        if it == 3:
            e0.record()
        rc = fn(ctypes.addressof(df.cfield), ctypes.addressof(dr.c), k, 0, hdr.block_grid[1], out.data_ptr(),
                hdr.height * hdr.width * 3, hdr.width * 3, status.data_ptr(), None)
        assert rc == 0
    e1.record()
    torch.cuda.synchronize()
    print(f"variant {extra}: last call {e0.elapsed_time(e1):.3f} ms")
    buf = np.zeros(64 * 8 * 8, dtype=np.int64)
    assert D.rlfc_dir_debug_times(buf.ctypes.data_as(ctypes.c_void_p)) == 0
    t = buf.reshape(64, 8, 8).astype(np.float64)
    names = ["wait inputs (cp.async + barrier)", "stage prefill (thread 0)", "phase A + barrier",
             "phase B + barrier", "phase C + barrier", "store + barrier", "tile total"]
    pairs = [(0, 1), (1, 2), (2, 3), (3, 4), (4, 5), (5, 6), (0, 6)]
    ok = t[:, :, 6] > 0
    for n, (a, b) in zip(names, pairs):
        d = ((t[:, :, b] - t[:, :, a]) / 1e3)[ok]
        print(f"{n:34s} median {np.median(d):7.3f} us  mean {d.mean():7.3f} us")


if __name__ == "__main__":
    main()
