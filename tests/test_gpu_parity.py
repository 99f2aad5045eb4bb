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
        for kern in ("auto", "dir", "staged", "fused", "simple"):
            got, _ = rl.decode_field(st, k, kernel=kern)
            assert sha(got.cpu().numpy()) == str(g[f"all_k{k}_sha"]), \
                (name, k, kern)
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


@pytest.mark.parametrize("kernel", ["dir", "staged", "fused"])
@pytest.mark.parametrize("name", ["mid17_r4", "b8_h2", "b16_h4", "odd_3x5",
                                  "kat8_default"])
def test_bands_and_subsets(rl, kernel, name):
    st = state_for(rl, name)
    full, _ = rl.decode_field(st, kernel="simple")
    full = full.cpu().numpy()
    S, T = st.header.s_count, st.header.t_count
    hb = st.header.block_grid[1]
    B = st.header.block_size
    for lo, hi in [(0, 3), (3, min(9, hb)), (min(9, hb), hb), (2, 2)]:
        lo, hi = min(lo, hb), min(hi, hb)
        for k in (0, 1):
            band, _ = rl.decode_field(st, k, rows=(lo, hi), kernel=kernel)
            ref, _ = rl.decode_field(st, k, rows=(lo, hi), kernel="simple")
            assert np.array_equal(band.cpu().numpy(), ref.cpu().numpy())
        band, _ = rl.decode_field(st, rows=(lo, hi), kernel=kernel)
        assert np.array_equal(band.cpu().numpy(),
                              full[:, :, lo * B:hi * B])
    imgs = [(S - 1, 0), (min(3, S - 1), min(2, T - 1)), (0, T - 1),
            (S // 2, T // 2)]
    imgs = list(dict.fromkeys(imgs))
    sub, _ = rl.decode_field(st, images=imgs, kernel=kernel)
    for i, (s, t) in enumerate(imgs):
        assert np.array_equal(sub[i].cpu().numpy(), full[s, t])
    sub, _ = rl.decode_field(st, images=imgs, rows=(1, min(4, hb)),
                             kernel=kernel)
    for i, (s, t) in enumerate(imgs):
        assert np.array_equal(sub[i].cpu().numpy(),
                              full[s, t, B:min(4, hb) * B])


@pytest.mark.parametrize("name", ["kat8_default", "mid17_r4", "b8_h2",
                                  "b16_h4", "grid32", "cfg1_h3_r4"])
def test_staged_path_taken(rl, name):
    """Inside its envelope the staged kernels really run (no silent
    fallback to the single-kernel path)."""
    import ctypes
    from paper_1805_06019_b200 import _native
    st = state_for(rl, name)
    df = st.device_field()
    ws, nbytes, present, nflag = df.staged_workspace(0)
    hdr = st.header
    out = torch.empty((hdr.s_count, hdr.t_count, hdr.height, hdr.width, 3),
                      dtype=torch.uint8, device="cuda")
    status = torch.zeros(1, dtype=torch.int64, device="cuda")
    rc = _native.lib().rlfc_decode_field_staged(
        df.ref, 0, None, 0, hdr.block_grid[1], out.data_ptr(),
        hdr.height * hdr.width * 3, hdr.width * 3, ws.data_ptr(), nbytes,
        present, nflag, None, 0, status.data_ptr(), 0)
    assert rc == _native.RLFC_OK
    torch.cuda.synchronize()
    assert status.item() == 0
    assert sha(out.cpu().numpy()) == str(load_golden(name)["all_k0_sha"])


@pytest.mark.parametrize("name", ["kat8_default", "mid17_r4", "grid32",
                                  "cfg1_h3_r4", "mid17_dense"])
def test_dir_path_taken(rl, name):
    """Inside its envelope the directory decode really runs: the ABI entry
    point accepts the stream and its output matches the reference golden."""
    from paper_1805_06019_b200 import _native
    st = state_for(rl, name)
    df = st.device_field()
    dr = df.directory()
    assert dr is not None and dr.n_flagged == 0
    hdr = st.header
    out = torch.empty((hdr.s_count, hdr.t_count, hdr.height, hdr.width, 3),
                      dtype=torch.uint8, device="cuda")
    status = torch.zeros(1, dtype=torch.int64, device="cuda")
    g = load_golden(name)
    for k in range(hdr.tree_height + 1):
        rc = _native.lib().rlfc_decode_field_dir(
            df.ref, dr.ref, k, 0, hdr.block_grid[1], out.data_ptr(),
            hdr.height * hdr.width * 3, hdr.width * 3, status.data_ptr(), 0)
        assert rc == _native.RLFC_OK
        torch.cuda.synchronize()
        assert status.item() == 0
        assert sha(out.cpu().numpy()) == str(g[f"all_k{k}_sha"]), k


@pytest.mark.parametrize("name", ["kat8_default", "mid17_r4", "b8_h2",
                                  "b16_h4", "alldesc_b4"])
def test_staged_fuzz_matches_simple(rl, name):
    """Random SRV corruptions: the staged path reports the same failure word
    (same key, same code) as the per-block kernel, and identical pixels when
    the reference would not raise."""
    from paper_1805_06019_b200 import container
    data = load_stream(name)
    hdr = container.parse_header(data)
    starts, _ = container.section_offsets(hdr)
    rng = np.random.default_rng(1234)
    agree = 0
    for trial in range(24):
        bad = bytearray(data)
        c = int(rng.integers(0, 3))
        lo = starts[c][2]
        n = hdr.section_lengths[c][2]
        for _ in range(int(rng.integers(1, 4))):
            pos = lo + int(rng.integers(0, n))
            bad[pos] = int(rng.integers(0, 256))
        st = rl.init(bytes(bad))
        for k in (0, hdr.tree_height - 1):
            b, sb = rl.decode_field(st, k, kernel="simple", check=False)
            for kern in ("dir", "staged"):
                a, sa = rl.decode_field(st, k, kernel=kern, check=False)
                assert sa.item() == sb.item(), (trial, k, kern)
                if sa.item() == 0:
                    assert np.array_equal(a.cpu().numpy(), b.cpu().numpy()), \
                        (trial, k, kern)
            agree += 1
    assert agree == 48


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
                for kern in ("dir", "staged", "fused", "simple"):
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


@pytest.mark.parametrize("name", ["kat8_default", "mid17_r4", "b8_h2", "odd_3x5", "b16_h4"])
def test_host_pipeline_matches_device_decode(rl, name):
    """decoder.HostPipeline (banded H2D | decode | D2H over three streams,
    the bench's e2e path) returns the same pixels as decode_field."""
    from paper_1805_06019_b200 import decoder
    st = state_for(rl, name)
    full, _ = rl.decode_field(st, kernel="simple")
    full = full.cpu().numpy()
    hb = st.header.block_grid[1]
    B = st.header.block_size
    for bands in (1, 3, 8):
        out = decoder.HostPipeline(st, bands=bands).run()
        assert np.array_equal(out.numpy(), full), bands
    lo, hi = (1, max(2, hb - 1)) if hb > 2 else (0, hb)
    out = decoder.HostPipeline(st, rows=(lo, hi), bands=2).run()
    assert np.array_equal(out.numpy(), full[:, :, lo * B:min(hi * B, st.header.height)])


@pytest.mark.parametrize("name", ["kat8_default", "mid17_r4"])
def test_corrupt_offsets_never_fault(rl, name):
    """Record offsets that leave the SRV section or run backwards (undefined
    in the reference, which does not bounds-check) must not fault the
    device: every kernel reports the same failure word, and decode_block
    raises FormatError or returns a block."""
    from paper_1805_06019_b200 import container
    data = load_stream(name)
    hdr = container.parse_header(data)
    starts, _ = container.section_offsets(hdr)
    wb, hb = hdr.block_grid
    rng = np.random.default_rng(99)
    for trial in range(6):
        bad = bytearray(data)
        c = int(rng.integers(0, 3))
        blk = int(rng.integers(1, wb * hb - 1))
        pos = starts[c][1] + 8 * blk
        val = [hdr.section_lengths[c][2] + 4096, 2 ** 40, 0, int(rng.integers(0, hdr.section_lengths[c][2]))][trial % 4]
        bad[pos:pos + 8] = int(val).to_bytes(8, "little")
        st = rl.init(bytes(bad))
        words = []
        for kern in ("dir", "staged", "fused", "simple"):
            _, sw = rl.decode_field(st, 0, kernel=kern, check=False)
            words.append(sw.item())
        assert len(set(words)) == 1, (trial, words)
        by, bx = divmod(blk, wb)
        try:
            rl.decode_block(st, (0, 0), (bx, by), c)
        except rl.FormatError:
            pass
    torch.cuda.synchronize()


@pytest.mark.parametrize("name", ["mid17_r4", "b8_h2", "b16_h4", "grid32", "mid17_dense"])
def test_indexed_random_access_matches_walk(rl, name):
    """Batches >= 4096 go through the prepared record index
    (rlfc_decode_blocks_indexed); values and codes equal the record walk's
    (rlfc_decode_blocks) for random picks at every stop level."""
    from paper_1805_06019_b200 import _native
    st = state_for(rl, name)
    hdr = st.header
    wb, hb = hdr.block_grid
    rng = np.random.default_rng(17)
    n = 6000
    req = np.stack([rng.integers(0, hdr.s_count, n), rng.integers(0, hdr.t_count, n),
                    rng.integers(0, wb, n), rng.integers(0, hb, n), rng.integers(-3, 3, n),
                    rng.integers(0, hdr.tree_height + 1, n)], 1).astype(np.int32)
    got, gst = rl.decode_blocks(st, req)
    df = st.device_field()
    dreq = torch.from_numpy(req % np.array([1 << 30] * 4 + [3, 1 << 30], np.int32)).cuda()
    want = torch.empty_like(got)
    wst = torch.zeros(n, dtype=torch.int32, device="cuda")
    assert _native.lib().rlfc_decode_blocks(df.ref, dreq.data_ptr(), n, want.data_ptr(), wst.data_ptr(), 0) == 0
    torch.cuda.synchronize()
    assert torch.equal(got, want) and torch.equal(gst, wst)
