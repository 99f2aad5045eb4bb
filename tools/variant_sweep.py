"""Time compile-time variants of the decode kernels on the cfg2 bench stream.

Measurement infrastructure only: each variant is the product library built
with extra -D flags into scratch/, loaded with ctypes beside the product
library (device memory is shared, so the DeviceField / workspace come from
the product path) and timed with CUDA events over the same call.

    python tools/variant_sweep.py [--preset R6] "-DRLFC_BLEND_BT=128 -DRLFC_BLEND_TW=128" ...

--preset picks a cfg2 bitrate preset (tools/bitrate_sweep.py PRESETS; the
stream is produced if missing), default R4 (the bench stream).
"""
import ctypes
import hashlib
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))


def build(flags):
    from paper_1805_06019_b200 import _build
    tag = hashlib.sha1(flags.encode()).hexdigest()[:8]
    out = os.path.join(ROOT, "scratch", f"libvariant_{tag}.so")
    cus = [os.path.join(_build.CSRC, f) for f in sorted(os.listdir(_build.CSRC)) if f.endswith(".cu")]
    subprocess.run(["nvcc"] + _build.NVCC_FLAGS + flags.split() + ["-o", out] + cus, check=True,
                   stderr=subprocess.DEVNULL)
    return out


def main():
    import torch
    import paper_1805_06019_b200 as rl
    from paper_1805_06019_b200 import _native
    import bench
    from bitrate_sweep import PRESETS
    args = sys.argv[1:]
    preset = "R4"
    if args[:1] == ["--preset"]:
        preset, args = args[1], args[2:]
    h, B, sh, tp, tb = PRESETS[preset]
    data, _ = bench.make_stream(dict(bench.CFG, h=h, B=B, shift=sh, tp=tp, tb=tb))
    st = rl.init(data)
    df = st.device_field()
    hdr = st.header
    out = torch.empty((hdr.s_count, hdr.t_count, hdr.height, hdr.width, 3), dtype=torch.uint8, device="cuda")
    status = torch.zeros(1, dtype=torch.int64, device="cuda")
    stream = torch.cuda.current_stream().cuda_stream
    ws = df.staged_workspace(stream)
    ref = rl.decode_field(st, 0, kernel="simple")[0].cpu()
    for flags in [""] + args:
        L = _native.load_library(build(flags)) if flags else _native.lib()
        # the variant library prepares its own copy of the workspace layout
        w2 = torch.empty_like(ws[0])
        nf = ctypes.c_int32(0)
        assert L.rlfc_staged_prepare(df.ref, w2.data_ptr(), ws[1], ws[2], ctypes.byref(nf), stream) == 0

        def call():
            return L.rlfc_decode_field_staged(df.ref, 0, None, 0, hdr.block_grid[1], out.data_ptr(),
                                              hdr.height * hdr.width * 3, hdr.width * 3, w2.data_ptr(), ws[1],
                                              ws[2], nf.value, None, 0, status.data_ptr(), stream)
        for _ in range(3):
            assert call() == 0
        torch.cuda.synchronize()
        ok = bool(torch.equal(out.cpu(), ref)) and status.item() == 0
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            call()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 20
        px = hdr.s_count * hdr.t_count * hdr.width * hdr.height
        print(f"{flags or 'product':50s} {ms:.4f} ms  {px / ms / 1e6:7.1f} Gpix/s  exact={ok}", flush=True)


if __name__ == "__main__":
    main()
