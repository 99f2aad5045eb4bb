"""Concurrency stress on one field (cfg2 R4 stream): 16 host threads mix
decode_block, decode_image, decode_plane, render_view and decode_blocks for
ROUNDS rounds while one thread runs decode_all; every result is compared
with a single-threaded reference computed first."""
import os
import sys
import threading

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1805_06019_b200 as rl  # noqa: E402
from paper_1805_06019_b200 import decoder  # noqa: E402

ROUNDS = int(os.environ.get("ROUNDS", "60"))
data, _ = bench.make_stream(bench.CFG)
st = rl.init(data)
rng = np.random.default_rng(3)
blocks = [((int(rng.integers(17)), int(rng.integers(17))), (int(rng.integers(256)), int(rng.integers(256))),
           int(rng.integers(3))) for _ in range(64)]
views = [(int(rng.integers(17)), int(rng.integers(17))) for _ in range(8)]
poses = [rl.SlabPose(float(rng.uniform(0, 16)), float(rng.uniform(0, 16)), 128, 128) for _ in range(8)]
ref_blocks = [rl.decode_block(st, *b) for b in blocks]
ref_images = [rl.decode_image(st, v) for v in views]
ref_planes = [rl.decode_plane(st, v[0], v[1], 1) for v in views]
ref_renders = [rl.render_view(st, p) for p in poses]
ref_all = rl.decode_all(st).rgb
errors = []


def worker(seed):
    r = np.random.default_rng(seed)
    try:
        for _ in range(ROUNDS):
            op = int(r.integers(5))
            i = int(r.integers(8))
            if op == 0:
                j = int(r.integers(64))
                assert np.array_equal(rl.decode_block(st, *blocks[j]), ref_blocks[j]), "block"
            elif op == 1:
                assert np.array_equal(rl.decode_image(st, views[i]), ref_images[i]), "image"
            elif op == 2:
                assert np.array_equal(rl.decode_plane(st, views[i][0], views[i][1], 1), ref_planes[i]), "plane"
            elif op == 3:
                assert np.array_equal(rl.render_view(st, poses[i]), ref_renders[i]), "render"
            else:
                req = np.array([[b[0][0], b[0][1], b[1][0], b[1][1], b[2], 0] for b in blocks], dtype=np.int32)
                out, _ = decoder.decode_blocks(st, req, raise_errors=False)
                got = out.cpu().numpy() if hasattr(out, "cpu") else np.asarray(out)
                assert np.array_equal(got.reshape(64, 4, 4), np.stack(ref_blocks)), "blocks"
    except Exception as exc:  # noqa: BLE001
        errors.append(repr(exc))


def all_worker():
    try:
        for _ in range(3):
            assert np.array_equal(rl.decode_all(st).rgb, ref_all), "decode_all"
    except Exception as exc:  # noqa: BLE001
        errors.append(repr(exc))


ths = [threading.Thread(target=worker, args=(s,)) for s in range(16)] + [threading.Thread(target=all_worker)]
for t in ths:
    t.start()
for t in ths:
    t.join()
torch.cuda.synchronize()
print("stress:", "ok" if not errors else f"{len(errors)} errors: {errors[:3]}", f"({16 * ROUNDS} mixed calls + 3 decode_all)")
