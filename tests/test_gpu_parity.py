"""GPU parity: the CUDA path (through the C ABI) against the reference goldens
and the C oracle.  Integer outputs and rendered views must be bit-exact."""
import json
import os

import numpy as np
import pytest

from conftest import GOLD, golden_names, load_golden, load_stream, sha

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

NAMES = golden_names()


@pytest.fixture(scope="module")
def rl():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1805_06019_b200 as rl
    return rl


_states = {}


def state_for(rl, name):
    if name not in _states:
        _states[name] = rl.init(load_stream(name))
    return _states[name]


@pytest.mark.parametrize("name", NAMES)
def test_decode_all_every_level(rl, name):
    g = load_golden(name)
    st = state_for(rl, name)
    for k in range(g["meta"]["h"] + 1):
        fused, _ = rl.decode_field(st, k)
        simple, _ = rl.decode_field(st, k, kernel="simple")
        f = fused.cpu().numpy()
        assert sha(f) == str(g[f"all_k{k}_sha"]), (name, k)
        assert np.array_equal(f, simple.cpu().numpy()), (name, k)
    grid = rl.decode_all(st)
    assert sha(grid.rgb) == str(g["all_k0_sha"])
    if "rgb_k0" in g:
        assert np.array_equal(grid.rgb, g["rgb_k0"])


@pytest.mark.parametrize("name", NAMES)
def test_decode_planes_every_level(rl, name):
    g = load_golden(name)
    st = state_for(rl, name)
    S, T = g["meta"]["S"], g["meta"]["T"]
    req = [(s, t, c) for s in range(S) for t in range(T) for c in range(3)]
    for k in range(g["meta"]["h"] + 1):
        planes = rl.decode_planes(st, req, k).cpu().numpy()
        hp, wp = planes.shape[1:]
        planes = planes.reshape(S, T, 3, hp, wp).astype("<i4")
        assert sha(planes) == str(g[f"planes_k{k}_sha"]), (name, k)


@pytest.mark.parametrize("name", NAMES)
def test_random_blocks(rl, name):
    g = load_golden(name)
    st = state_for(rl, name)
    out, status = rl.decode_blocks(st, g["blocks_req"])
    assert np.array_equal(out.cpu().numpy(), g["blocks_val"])
    assert not status.cpu().numpy().any()
    for (s, t, bx, by, c, k), want in list(zip(g["blocks_req"],
                                               g["blocks_val"]))[:10]:
        got = rl.decode_block_progressive(st, (int(s), int(t)),
                                          (int(bx), int(by)), int(c), int(k))
        assert got.dtype == np.int32 and np.array_equal(got, want)


def _pose(rl, p):
    if p["kind"] == "slab":
        return rl.SlabPose(p["s"], p["t"], p["width"], p["height"],
                           p["focal_z"])
    return rl.CameraPose(tuple(p["eye"]), tuple(p["look"]), p["fov_deg"],
                         p["width"], p["height"])


@pytest.mark.parametrize("name", NAMES)
def test_render_views_bit_exact(rl, name):
    g = load_golden(name)
    st = state_for(rl, name)
    for i, r in enumerate(g["meta"]["renders"]):
        geo = r.get("geometry")
        geometry = None if geo is None else rl.PlaneGeometry(
            geo[0], geo[1], tuple(geo[2]))
        out = rl.render_view(st, _pose(rl, r["pose"]), stop_level=r["k"],
                             geometry=geometry,
                             background=tuple(r["background"]))
        assert np.array_equal(out, g[f"render_{i}"]), (name, i, r)


def test_render_batch_equals_single(rl):
    st = state_for(rl, "mid17_r4")
    rng = np.random.default_rng(3)
    poses = [rl.SlabPose(float(rng.uniform(0, 16)), float(rng.uniform(0, 16)),
                         32, 32) for _ in range(12)]
    batch = rl.render_views(st, poses).cpu().numpy()
    for p, img in zip(poses, batch):
        assert np.array_equal(img, rl.render_view(st, p))


def test_bands_and_subsets(rl):
    st = state_for(rl, "mid17_r4")
    full, _ = rl.decode_field(st)
    full = full.cpu().numpy()
    hb = st.header.block_grid[1]
    B = st.header.block_size
    for lo, hi in [(0, 3), (3, 9), (9, hb), (5, 5)]:
        band, _ = rl.decode_field(st, rows=(lo, hi))
        assert np.array_equal(band.cpu().numpy(),
                              full[:, :, lo * B:hi * B])
    imgs = [(16, 0), (3, 7), (0, 16), (8, 8)]
    sub, _ = rl.decode_field(st, images=imgs)
    for i, (s, t) in enumerate(imgs):
        assert np.array_equal(sub[i].cpu().numpy(), full[s, t])


def test_corrupt_streams_raise_like_reference(rl):
    with open(os.path.join(GOLD, "corrupt.json")) as f:
        cases = json.load(f)
    for case in cases:
        st = rl.init(load_stream(case["name"]))
        for call in case["calls"]:
            parts = call["call"].split()
            args = list(map(int, parts[1:]))

            def run():
                if parts[0] == "decode_block":
                    s, t, bx, by, c, k = args
                    return rl.decode_block_progressive(st, (s, t), (bx, by),
                                                       c, k)
                if parts[0] == "decode_plane":
                    s, t, c, k = args
                    return rl.decode_plane(st, s, t, c, k)
                if parts[0] == "decode_image":
                    s, t, k = args
                    from paper_1805_06019_b200 import decoder
                    return decoder.decode_image(st, (s, t), k)
                for kern in ("fused", "simple"):
                    rl.decode_field(st, args[0], kernel=kern)
                return rl.decode_all(st, args[0])
            if call["exc"] is None:
                run()
            else:
                with pytest.raises(rl.FormatError) as ei:
                    run()
                assert str(ei.value) == {
                    "corrupt coded pack in SRV payload":
                        "corrupt coded pack in SRV payload",
                    "descriptor outside range table":
                        "descriptor outside range table"}[call["msg"]], call


def test_bise_decode_vectors(rl):
    from paper_1805_06019_b200 import bise, decoder
    z = np.load(os.path.join(GOLD, "bise_vectors.npz"))
    payload, index, values = z["payload"], z["index"], z["values"]
    pos = 0
    for count in sorted(set(int(n) for n in index[:, 1])):
        rows = [(i, r) for i, r in enumerate(index) if r[1] == count]
        blobs = [payload[r[2]:r[2] + r[3]].tobytes() for _, r in rows]
        vals, status = decoder.bise_decode_batch(blobs, [r[0] for _, r in rows],
                                                 count)
        assert not status.any()
        starts = np.cumsum([0] + [int(r[1]) for r in index])
        for j, (i, r) in enumerate(rows):
            assert np.array_equal(vals[j], values[starts[i]:starts[i] + count])
    assert bise.bise_decode(bytes([0x0B, 0x05]), 3,
                            bise.RANGE_TABLE[4]).tolist() == [5, 0, 3]
    with pytest.raises(rl.FormatError):
        bise.bise_decode(bytes([243]), 5, bise.RANGE_TABLE[1])
    with pytest.raises(rl.FormatError):
        bise.bise_decode(bytes([125]), 3, bise.RANGE_TABLE[3])


def test_gpu_matches_oracle_random_access(rl):
    from oracle import oracle
    for name in ("grid32", "alldesc_b4", "mid17_dense"):
        data = load_stream(name)
        st = state_for(rl, name)
        orc = oracle.OracleState(data)
        rng = np.random.default_rng(5)
        hdr = st.header
        wb, hb = hdr.block_grid
        req = np.stack([rng.integers(0, hdr.s_count, 500),
                        rng.integers(0, hdr.t_count, 500),
                        rng.integers(0, wb, 500), rng.integers(0, hb, 500),
                        rng.integers(0, 3, 500),
                        rng.integers(0, hdr.tree_height + 1, 500)], 1)
        out, _ = rl.decode_blocks(st, req)
        out = out.cpu().numpy()
        for r, got in zip(req, out):
            want, code = orc.decode_block(*map(int, r))
            assert code == 0 and np.array_equal(got, want)
