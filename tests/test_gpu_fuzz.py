"""Seeded configuration fuzz over the format's parameter space (GPU).

Random small fields -- grid sizes 1..24, odd image sizes (some wider than
two 64-pixel blend chunks), B in {2, 4, 8, 16}, tree heights 1..5,
quantiser shifts 0..8 (int16 and int32 residuals), pixel /
block thresholds from lossless to coarse, both filters, RAW and PNG roots --
are synthesised and encoded twice: by the native C++ producer and by the GPU
tree construction, which must agree byte for byte (the producer is pinned to
the reference encoder by tests/test_producer.py).  Every decode kernel, image
subsets, block-row bands, random blocks, a slab and a pinhole render are then compared
with the C oracle (pinned to the reference by tests/test_oracle_golden.py) at
several stop levels.  Integer outputs bit-exact, renders bit-exact.
"""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


MAXST = int(os.environ.get("FUZZ_MAXST", "24"))
MAXH = int(os.environ.get("FUZZ_MAXH", "5"))
MAXSHIFT = int(os.environ.get("FUZZ_MAXSHIFT", "8"))


def _configs(n=64, seed=2026):
    rng = np.random.default_rng(seed)
    out = []
    for i in range(n):
        B = int(rng.choice([2, 4, 8, 16], p=[0.15, 0.45, 0.25, 0.15]))
        h = int(rng.integers(1, MAXH + 1))
        big = i % 4 == 3                       # every fourth: wide images (several 64-pixel blend chunks)
        S, T = int(rng.integers(1, MAXST + 1)), int(rng.integers(1, MAXST + 1))
        W = int(rng.integers(130, 300)) if big else int(rng.integers(max(2, B // 2), 72))
        H = int(rng.integers(max(2, B // 2), 72))
        shift = int(rng.integers(0, MAXSHIFT + 1))
        tp = int(rng.choice([0, 1, 2, 4, 8, 16, 32]))
        tb = int(rng.choice([0, 10, 80, 300, 1000]))
        filt = str(rng.choice(["gaussian", "uniform"]))
        codec = str(rng.choice(["raw", "png"]))
        out.append(dict(spec=dict(s_count=S, t_count=T, width=W, height=H, seed=int(rng.integers(0, 1000))),
                        params=dict(tree_height=h, block_size=B, quant_shift=shift, pixel_threshold=tp,
                                    block_threshold=tb, filter=filt, root_codec=codec)))
    return out


# extended hunts: FUZZ_N=1000 FUZZ_SEED=7 python -m pytest tests/test_gpu_fuzz.py
CONFIGS = _configs(int(os.environ.get("FUZZ_N", "64")), int(os.environ.get("FUZZ_SEED", "2026")))


@pytest.fixture(scope="module")
def rl():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1805_06019_b200 as rl
    return rl


@pytest.mark.parametrize("i", range(len(CONFIGS)))
def test_config_fuzz(rl, i):
    from oracle import oracle
    from paper_1805_06019_b200 import decoder, encoder, lightfield, producer
    cfg = CONFIGS[i]
    p = dict(cfg["params"])
    p["filter"] = encoder.FilterSpec(kind=p["filter"])
    params = encoder.EncodingParams(**p)
    lf = lightfield.synthesize_lightfield(lightfield.SyntheticSpec(**cfg["spec"]))
    data, present = producer.encode(lf, params)
    gdata, gpresent = producer.encode_gpu(lf, params)
    assert gdata == data and tuple(gpresent) == tuple(present), cfg
    st = rl.init(data)
    orc = oracle.OracleState(data)
    hdr = st.header
    S, T, h = hdr.s_count, hdr.t_count, hdr.tree_height
    wb, hb = hdr.block_grid
    rng = np.random.default_rng(100 + i)
    for k in sorted({0, h // 2, h}):
        want, code = orc.decode_all(k)
        assert code == 0
        for kernel in ("auto", "dir", "fused", "simple"):
            got, _ = decoder.decode_field(st, k, kernel=kernel)
            assert np.array_equal(got.cpu().numpy(), want), (cfg, k, kernel)
        # a subset of views (slot mode) over a block-row band
        n_img = int(rng.integers(1, S * T + 1))
        picks = [tuple(map(int, divmod(int(j), T))) for j in rng.choice(S * T, n_img, replace=False)]
        lo = int(rng.integers(0, hb))
        hi = int(rng.integers(lo + 1, hb + 1))
        got, _ = decoder.decode_field(st, k, images=picks, rows=(lo, hi))
        r0, r1 = lo * hdr.block_size, min(hi * hdr.block_size, hdr.height)
        for j, (s, t) in enumerate(picks):
            assert np.array_equal(got[j].cpu().numpy(), want[s, t, r0:r1]), (cfg, k, (s, t), (lo, hi))
    # 64 requests take the per-request walk, 4096 the prepared-index path
    for nreq in (64, 4096):
        req = np.stack([rng.integers(0, S, nreq), rng.integers(0, T, nreq), rng.integers(0, wb, nreq),
                        rng.integers(0, hb, nreq), rng.integers(0, 3, nreq), rng.integers(0, h + 1, nreq)], 1)
        out, _ = rl.decode_blocks(st, req)
        out = out.cpu().numpy()
        for r, blk in zip(req, out):
            want, code = orc.decode_block(*map(int, r))
            assert code == 0 and np.array_equal(blk, want), (cfg, nreq, r)
    s, t = float(rng.uniform(0, S - 1)), float(rng.uniform(0, T - 1))
    focal = [None, 0.9, 1.12][i % 3]
    k = int(rng.integers(0, h + 1))
    img = rl.render_view(st, rl.SlabPose(s, t, 24, 20, focal_z=focal), stop_level=k)
    assert np.array_equal(img, orc.render_slab(s, t, 24, 20, focal_z=focal, stop_level=k)), (cfg, s, t, focal, k)
    eye = (float(rng.uniform(-1, S)), float(rng.uniform(-1, T)), -float(rng.uniform(1, 4)))
    look = (float(rng.uniform(-0.2, 0.2)), float(rng.uniform(-0.2, 0.2)), 1.0)
    img = rl.render_view(st, rl.CameraPose(eye=eye, look=look, fov_deg=40.0, width=16, height=12), stop_level=k)
    want = orc.render_pinhole(eye, look, 40.0, 16, 12, stop_level=k)
    want = want[0] if isinstance(want, tuple) else want
    assert np.array_equal(img, want), (cfg, eye, look, k)


def _walk_past_end(data, hdr, c, s, t, bx, by, k):
    """True when the reference-order walk of record (c, bx, by) for view
    (s, t) down to level k (kernels.py:162-216: node by node, descriptor +
    payload sizes) runs past the end of channel c's SRV section before it
    meets an out-of-table descriptor."""
    from paper_1805_06019_b200 import bise, container
    from oracle.oracle import chains_for
    S, T, h, B = hdr.s_count, hdr.t_count, hdr.tree_height, hdr.block_size
    wb, hb = hdr.block_grid
    starts, _ = container.section_offsets(hdr)
    offs = np.frombuffer(data, dtype="<u8", count=wb * hb, offset=starts[c][1])
    sec0, sec1 = starts[c][2], starts[c][2] + hdr.section_lengths[c][2]
    targets = chains_for(S, T, h)[s, t][:h - k]
    if len(targets) == 0:
        return False
    m = sum(container.level_dims(S, T, l)[0] * container.level_dims(S, T, l)[1] for l in range(h))
    rec = sec0 + int(offs[by * wb + bx])
    nbm = (m + 7) // 8
    if rec + nbm > sec1:
        return True
    cur = rec + nbm
    for node in range(int(targets[-1]) + 1):
        if not (data[rec + (node >> 3)] >> (node & 7)) & 1:
            continue
        if cur >= sec1:
            return True
        d = data[cur]
        if d >= len(bise.RANGE_TABLE):
            return False
        r = bise.RANGE_TABLE[d]
        size = 1 + (bise.payload_bits(r.mode, r.low_bits, B * B) + 7) // 8
        if cur + size > sec1:
            return True
        cur += size
    return False


@pytest.mark.parametrize("i", range(0, len(CONFIGS), 2))
def test_corrupt_fuzz(rl, i):
    """Random byte corruptions of the SRV sections of the fuzz fields: the
    whole-field decode (staged and per-block kernels) fails exactly when the
    oracle's reference-order decode_all fails, with the same code -- hence
    the same FormatError -- and otherwise returns the oracle's pixels; random
    blocks report the oracle's per-block codes."""
    from oracle import oracle
    from paper_1805_06019_b200 import _native, container, decoder, encoder, lightfield, producer
    cfg = CONFIGS[i]
    p = dict(cfg["params"])
    p["filter"] = encoder.FilterSpec(kind=p["filter"])
    lf = lightfield.synthesize_lightfield(lightfield.SyntheticSpec(**cfg["spec"]))
    data, _ = producer.encode(lf, encoder.EncodingParams(**p))
    hdr = container.parse_header(data)
    starts, _ = container.section_offsets(hdr)
    rng = np.random.default_rng(500 + i)
    for trial in range(3):
        c = int(rng.integers(0, 3))
        n = hdr.section_lengths[c][2]
        if n == 0:
            continue
        bad = bytearray(data)
        for _ in range(int(rng.integers(1, 4))):
            bad[starts[c][2] + int(rng.integers(0, n))] = int(rng.integers(0, 256))
        bad = bytes(bad)
        st = rl.init(bad)
        orc = oracle.OracleState(bad)
        wb, hb = hdr.block_grid
        for k in sorted({0, hdr.tree_height - 1}):
            want, wcode = orc.decode_all(k)
            for kernel in ("auto", "simple"):
                got, status = decoder.decode_field(st, k, kernel=kernel, check=False)
                word = _native.decode_status_word(status.item())
                gcode = 0 if word is None else word[1]
                if gcode == 2 and wcode != 2:
                    key = word[0]
                    blk, ic = key % (wb * hb), key // (wb * hb)
                    img, cc = divmod(ic, 3)
                    if _walk_past_end(bad, hdr, cc, img // hdr.t_count, img % hdr.t_count, blk % wb, blk // wb, k):
                        # the walk ran past the SRV section's end: the
                        # reference reads out of bounds there (numba does not
                        # bounds-check; its Python backend raises IndexError),
                        # the oracle reads its zero tail, this decoder reports
                        # code 2 ((c))
                        break
                assert gcode == wcode, (cfg, trial, k, kernel)
                if wcode == 0:
                    assert np.array_equal(got.cpu().numpy(), want), (cfg, trial, k, kernel)
        S, T = hdr.s_count, hdr.t_count
        # single images (decoder.py:187-194: planes of channels 0, 1, 2, the
        # first failing one raises) and single planes, through the one-call
        # host paths
        for _ in range(3):
            s, t = int(rng.integers(0, S)), int(rng.integers(0, T))
            k = int(rng.integers(0, hdr.tree_height))
            codes = [orc.decode_plane(s, t, cc, k)[1] for cc in range(3)]
            want_code = next((x for x in codes if x), 0)
            try:
                img = rl.decode_image(st, (s, t), stop_level=k)
                got_code = 0
            except rl.FormatError as e:
                got_code = 2 if "descriptor" in str(e) else 1
                img = None
            if got_code != want_code:
                assert got_code == 2 and any(
                    _walk_past_end(bad, hdr, cc, s, t, bx, by, k)
                    for cc in range(3) for by in range(hb) for bx in range(wb)), (cfg, trial, s, t, k)
            elif want_code == 0:
                want_img, _ = orc.decode_all(k)
                assert np.array_equal(img, want_img[s, t]), (cfg, trial, s, t, k)
            cc = int(rng.integers(0, 3))
            wplane, wcode = orc.decode_plane(s, t, cc, k)
            try:
                plane = rl.decode_plane(st, s, t, cc, stop_level=k)
                pcode = 0
            except rl.FormatError as e:
                pcode = 2 if "descriptor" in str(e) else 1
            if pcode != wcode:
                assert pcode == 2 and any(_walk_past_end(bad, hdr, cc, s, t, bx, by, k)
                                          for by in range(hb) for bx in range(wb)), (cfg, trial, s, t, cc, k)
            elif wcode == 0:
                assert np.array_equal(plane, wplane), (cfg, trial, s, t, cc, k)
        req = np.stack([rng.integers(0, S, 32), rng.integers(0, T, 32), rng.integers(0, wb, 32),
                        rng.integers(0, hb, 32), np.full(32, c), rng.integers(0, hdr.tree_height + 1, 32)], 1)
        out, status = rl.decode_blocks(st, req, raise_errors=False)
        out, status = out.cpu().numpy(), status.cpu().numpy()
        for r, blk, code in zip(req, out, status):
            want, wcode = orc.decode_block(*map(int, r))
            if int(code) == 2 and wcode != 2 and _walk_past_end(bad, hdr, int(r[4]), int(r[0]), int(r[1]),
                                                                 int(r[2]), int(r[3]), int(r[5])):
                continue                          # past the section end, as above
            assert int(code) == int(wcode), (cfg, trial, r)
            if wcode == 0:
                assert np.array_equal(blk, want), (cfg, trial, r)
