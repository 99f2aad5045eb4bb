"""Host-side logic on CPU: container parsing, BFS geometry, range table,
locate_block, error behaviour of init-time parsing (no GPU needed)."""
import json
import os
import struct

import numpy as np
import pytest

from conftest import GOLD, golden_names, load_golden, load_stream, sha

from paper_1805_06019_b200 import bise, container
from paper_1805_06019_b200.errors import FormatError, UnsupportedCodecError
from oracle import oracle


def test_range_table_matches_reference_constants():
    # test_bise.py:17-49 of the reference
    assert bise.RANGE_CARDINALITIES == (
        2, 3, 4, 5, 6, 8, 10, 12, 16, 20, 24, 32, 40, 48, 64, 80, 96, 128,
        160, 192, 256, 320, 384, 512, 640, 768, 1024, 1280, 1536, 2048)
    head = [(e.cardinality, e.mode, e.low_bits) for e in bise.RANGE_TABLE[:8]]
    assert head == [(2, 0, 1), (3, 1, 0), (4, 0, 2), (5, 2, 0), (6, 1, 1),
                    (8, 0, 3), (10, 2, 1), (12, 1, 2)]
    assert bise.select_range(255).cardinality == 256
    assert bise.select_range(256).cardinality == 320
    with pytest.raises(FormatError):
        bise.select_range(2048)
    # Appendix A payload bytes at B=4
    assert bise.payload_bytes_table(16).tolist() == [
        2, 4, 4, 6, 6, 6, 8, 8, 8, 10, 10, 10, 12, 12, 12, 14, 14, 14, 16,
        16, 16, 18, 18, 18, 20, 20, 20, 22, 22, 22]


@pytest.mark.parametrize("name", golden_names())
def test_header_sections_chains(name):
    g = load_golden(name)
    meta = g["meta"]
    data = load_stream(name)
    hdr = container.parse_header(data)
    container.check_stream_length(hdr, data)
    assert (hdr.s_count, hdr.t_count, hdr.width, hdr.height) == (
        meta["S"], meta["T"], meta["W"], meta["H"])
    assert hdr.block_size == meta["B"] and hdr.tree_height == meta["h"]
    assert [list(s) for s in hdr.section_lengths] == meta["sections"]
    assert container.total_srv_nodes(hdr.s_count, hdr.t_count,
                                     hdr.tree_height) == meta["m_nodes"]
    chains = container.all_chains(hdr.s_count, hdr.t_count, hdr.tree_height)
    assert np.array_equal(chains, g["chains"])
    for s, t in [(0, 0), (hdr.s_count - 1, hdr.t_count - 1)]:
        assert np.array_equal(container.chain_node_indices(
            s, t, hdr.s_count, hdr.t_count, hdr.tree_height), chains[s, t])
    roots = container.parse_roots(data, hdr)
    assert sha(roots.astype(np.int32)) == str(g["root_planes_sha"])
    assert container.pack_header(hdr) == data[:64]


def test_bfs_kats():
    # reference test_container.py:101-149 style known answers (8x8, h=3)
    assert container.level_dims(8, 8, 1) == (4, 4)
    assert container.level_dims(17, 17, 2) == (5, 5)
    assert container.level_node_counts(8, 8, 3) == [64, 16, 4]
    assert container.bfs_index(2, 0, 0, 8, 8, 3) == 0
    assert container.bfs_index(1, 0, 0, 8, 8, 3) == 4
    assert container.bfs_index(0, 7, 7, 8, 8, 3) == 83
    assert container.chain_node_indices(5, 2, 8, 8, 3).tolist() == [1, 10, 41]
    with pytest.raises(ValueError):
        container.bfs_index(3, 0, 0, 8, 8, 3)


def test_locate_block_agrees_with_oracle_walk():
    data = load_stream("mid17_r4")
    hdr = container.parse_header(data)
    st = oracle.OracleState(data)
    rng = np.random.default_rng(1)
    wb, hb = hdr.block_grid
    for _ in range(100):
        c = int(rng.integers(0, 3))
        blk = int(rng.integers(0, wb * hb))
        node = int(rng.integers(0, st.m_nodes))
        got = container.locate_block(data, hdr, c, blk, node)
        rec = int(st.offsets[c][blk])
        bits = np.unpackbits(st.srv[c][rec:rec + (st.m_nodes + 7) // 8],
                             bitorder="little")
        assert (got is None) == (not bits[node])


def test_header_errors_match_reference():
    data = bytearray(load_stream("kat8_default"))
    with pytest.raises(FormatError):
        container.parse_header(b"garbage")
    bad = bytearray(data)
    bad[:4] = b"XXXX"
    with pytest.raises(FormatError, match="magic"):
        container.parse_header(bytes(bad))
    bad = bytearray(data)
    bad[5] = 9
    with pytest.raises(UnsupportedCodecError):
        container.parse_header(bytes(bad))
    bad = bytearray(data)
    bad[6] = 3
    with pytest.raises(FormatError, match="block size"):
        container.parse_header(bytes(bad))
    hdr = container.parse_header(bytes(data))
    with pytest.raises(FormatError, match="truncated"):
        container.check_stream_length(hdr, bytes(data[:100]))
    with pytest.raises(FormatError, match="trailing"):
        container.check_stream_length(hdr, bytes(data) + b"\0")


def test_balanced_bands_partition_rows():
    from paper_1805_06019_b200 import parallel

    class St:
        pass
    data = load_stream("mid17_r4")
    st = St()
    st.header = container.parse_header(data)
    st.offsets = tuple(container.parse_offsets(data, st.header, c)
                       for c in range(3))
    hb = st.header.block_grid[1]
    for n in (1, 2, 3, 4, 8):
        bands = parallel.balanced_bands(st, n)
        assert len(bands) == n and bands[0][0] == 0 and bands[-1][1] == hb
        assert all(a[1] == b[0] for a, b in zip(bands, bands[1:]))
        cost = parallel.row_costs(st)
        per = [cost[lo:hi].sum() for lo, hi in bands]
        assert max(per) <= cost.sum() / n + cost.max() + 1e-6


def test_parallel_root_parse_matches_serial():
    """container.parse_roots decodes the root images on a thread pool; values
    and the first error in stream order are those of the plane-by-plane walk
    (container.py:355-379)."""
    import struct
    from paper_1805_06019_b200 import container
    from paper_1805_06019_b200.errors import FormatError
    data = load_stream("kat8_default")
    hdr = container.parse_header(data)
    assert hdr.root_codec_id == container.CODEC_PNG
    a = container.parse_roots(data, hdr, threads=1)
    b = container.parse_roots(data, hdr, threads=8)
    assert np.array_equal(a, b)
    starts, _ = container.section_offsets(hdr)
    # corrupt the image bytes of the first root plane of channel 1
    pos = starts[1][0]
    n = struct.unpack_from("<I", data, pos)[0]
    bad = bytearray(data)
    bad[pos + 4 + 8:pos + 4 + 24] = b"\xff" * 16
    msgs = []
    for th in (1, 8):
        with pytest.raises(FormatError) as ei:
            container.parse_roots(bytes(bad), hdr, threads=th)
        msgs.append(str(ei.value))
    import re
    strip = [re.sub(r" at 0x[0-9a-f]+", "", m) for m in msgs]      # object addresses
    assert strip[0] == strip[1] and "decode failed" in strip[0]
    # ... and also make channel 2's root length run past its section: the
    # earlier decode error still comes first
    pos2 = starts[2][0]
    bad[pos2:pos2 + 4] = struct.pack("<I", 1 << 30)
    for th in (1, 8):
        with pytest.raises(FormatError, match="decode failed"):
            container.parse_roots(bytes(bad), hdr, threads=th)
    only_trunc = bytearray(data)
    only_trunc[pos2:pos2 + 4] = struct.pack("<I", 1 << 30)
    for th in (1, 8):
        with pytest.raises(FormatError, match="truncated"):
            container.parse_roots(bytes(only_trunc), hdr, threads=th)
    assert n > 24


def test_colour_kat():
    """test_colorspace.py:9-11: (255, 0, 0) <-> YCoCg-R (63, 255, -127)."""
    from paper_1805_06019_b200 import colorspace
    y, co, cg = colorspace.rgb_to_ycocgr(np.array([255]), np.array([0]), np.array([0]))
    assert (int(y[0]), int(co[0]), int(cg[0])) == (63, 255, -127)
    r, g, b = colorspace.ycocgr_to_rgb(y, co, cg)
    assert (int(r[0]), int(g[0]), int(b[0])) == (255, 0, 0)


def test_request_range_checks():
    """decoder._check_requests mirrors decoder.py:51-63 for batched
    requests and normalises Python-style negative channels."""
    from paper_1805_06019_b200 import container, decoder

    class St:
        pass
    st = St()
    st.header = container.parse_header(load_stream("mid17_r4"))
    wb, hb = st.header.block_grid
    ok = np.array([[0, 0, 0, 0, -1, 0], [16, 16, wb - 1, hb - 1, 2, 3]], np.int32)
    out = decoder._check_requests(st, ok, 6)
    assert out[0, 4] == 2 and ok[0, 4] == -1
    for col, val, exc in [(0, 17, IndexError), (1, -1, IndexError), (2, wb, IndexError),
                          (3, -1, IndexError), (4, 3, IndexError), (4, -4, IndexError), (5, 4, ValueError)]:
        bad = ok.copy()
        bad[1, col] = val
        with pytest.raises(exc):
            decoder._check_requests(st, bad, 6)
    with pytest.raises(IndexError):
        decoder._check_requests(st, np.array([[0, 0, 3]], np.int32), 3)
