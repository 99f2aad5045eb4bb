"""W >= 256 fields against the live reference (tests/golden/large.json).

CPU: the native producer regenerates the reference's streams byte for byte,
and the C oracle decodes them to the reference's decode_all sha256 at every
stop level (pins the oracle beyond the W <= 64 goldens).
GPU: every decode kernel matches the reference's decode_all sha256 at every
stop level (B = 4 at W = 256 runs >= 4 column chunks per blend row; B = 8 and
B = 16 at 512^2), random blocks match, and 512x512 slab renders (focal at
the image plane, 0.9, 1.12; k = 0 and 2) match the reference renders; the
full cfg2 R4 field (17x17x1024^2, the bench workload) matches the
reference's decode_all sha256 (tests/golden/cfg2_r4_decode_reference.json).
"""
import hashlib
import json
import os

import numpy as np
import pytest

from conftest import GOLD
from large_fields import cfg2_stream, golden, stream

NAMES = sorted(golden())


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.mark.parametrize("name", NAMES)
def test_producer_reproduces_reference_stream(name):
    assert len(stream(name)) == golden()[name]["stream_bytes"]


@pytest.mark.parametrize("name", ["w256_r4", "w512_b8"])
def test_oracle_matches_reference_decode(name):
    from oracle import oracle
    g = golden()[name]
    orc = oracle.OracleState(stream(name))
    for k in range(g["h"] + 1):
        out, st = orc.decode_all(k, nthreads=oracle.lib().orc_nproc())
        assert st == 0 and _sha(out) == g[f"all_k{k}_sha"], (name, k)


@pytest.fixture(scope="module")
def rl():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1805_06019_b200 as rl
    return rl


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_gpu_decode_matches_reference(rl, name):
    g = golden()[name]
    st = rl.init(stream(name))
    for k in range(g["h"] + 1):
        for kern in ("auto", "staged", "dir", "fused"):
            out, _ = rl.decode_field(st, k, kernel=kern)
            assert _sha(out.cpu().numpy()) == g[f"all_k{k}_sha"], (name, k, kern)
    for s, t, bx, by, c, k, vals in g["blocks"]:
        got = rl.decode_block_progressive(st, (s, t), (bx, by), c, k)
        assert got.ravel().tolist() == vals


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_gpu_render_512_matches_reference(rl, name):
    g = golden()[name]
    st = rl.init(stream(name))
    poses = []
    for r in g["renders"]:
        pose = rl.SlabPose(r["s"], r["t"], 512, 512, r["focal_z"])
        img = rl.render_view(st, pose, stop_level=r["k"])
        assert _sha(img) == r["sha256"], r
        if r["k"] == 0:
            poses.append((pose, r["sha256"]))
    # the batched path (one tap-camera decode, one render launch)
    batch = rl.render_views(st, [p for p, _ in poses]).cpu().numpy()
    for img, (_, want) in zip(batch, poses):
        assert _sha(img) == want


@pytest.mark.gpu
def test_gpu_cfg2_r4_matches_reference(rl):
    with open(os.path.join(GOLD, "cfg2_r4_decode_reference.json")) as f:
        want = json.load(f)
    st = rl.init(cfg2_stream())
    for k in (0, 3):
        out, _ = rl.decode_field(st, k)
        assert _sha(out.cpu().numpy()) == want[f"k{k}"]["decode_all_sha256"], k
