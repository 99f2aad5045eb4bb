"""Route 2: the reference's kernel-module entry points with
their own argument tuples, run on the GPU by kernels_b200.py.  Arguments are
built exactly as the reference decoder builds them (decoder.py:81-106 for
decode_chain_core, decoder.py:165-184 for decode_plane_core); results must
equal the reference goldens."""
import numpy as np
import pytest

from conftest import GOLD, golden_names, load_golden, load_stream, sha

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def kb():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1805_06019_b200 import kernels_b200
    return kernels_b200


def _state(name):
    from paper_1805_06019_b200 import container
    data = load_stream(name)
    hdr = container.parse_header(data)
    roots = container.parse_roots(data, hdr)
    offs = [container.parse_offsets(data, hdr, c) for c in range(3)]
    srv = [np.frombuffer(container.srv_section(data, hdr, c), dtype=np.uint8) for c in range(3)]
    chains = container.all_chains(hdr.s_count, hdr.t_count, hdr.tree_height)
    m = container.total_srv_nodes(hdr.s_count, hdr.t_count, hdr.tree_height)
    return hdr, roots, offs, srv, chains, m


TABLE_MODE = np.array([r.mode for r in __import__("paper_1805_06019_b200.bise", fromlist=["x"]).RANGE_TABLE], np.uint8)
TABLE_BITS = np.array([r.low_bits for r in __import__("paper_1805_06019_b200.bise", fromlist=["x"]).RANGE_TABLE],
                      np.uint8)


@pytest.mark.parametrize("name", ["kat8_default", "mid17_r4", "b8_h2", "b16_h4", "alldesc_b4", "b2_h1"])
def test_decode_chain_core_matches_golden_blocks(kb, name):
    g = load_golden(name)
    hdr, roots, offs, srv, chains, m = _state(name)
    B, h = hdr.block_size, hdr.tree_height
    wb = hdr.block_grid[0]
    for (s, t, bx, by, c, k), want in list(zip(g["blocks_req"], g["blocks_val"]))[:40]:
        s, t, bx, by, c, k = map(int, (s, t, bx, by, c, k))
        out = roots[s >> h, t >> h, c, by * B:(by + 1) * B, bx * B:(bx + 1) * B].astype(np.int32).reshape(-1).copy()
        targets = chains[s, t, :h - k]
        tmp = np.empty(B * B, np.uint32)
        st = kb.decode_chain_core(srv[c], int(offs[c][by * wb + bx]), m, B * B, targets, hdr.quant_shift,
                                  TABLE_MODE, TABLE_BITS, out, tmp)
        assert st == 0 and np.array_equal(out.reshape(B, B), want)


@pytest.mark.parametrize("name", ["kat8_default", "mid17_r4", "odd_3x5", "b16_h4"])
def test_decode_plane_core_matches_golden_planes(kb, name):
    g = load_golden(name)
    hdr, roots, offs, srv, chains, m = _state(name)
    h, B = hdr.tree_height, hdr.block_size
    wb, hb = hdr.block_grid
    S, T = hdr.s_count, hdr.t_count
    for k in (0, h - 1):
        planes = np.zeros((S, T, 3) + roots.shape[3:], np.int32)
        for s in range(S):
            for t in range(T):
                for c in range(3):
                    out = np.empty(roots.shape[3:], np.int32)
                    st = kb.decode_plane_core(srv[c], offs[c], wb, hb, m, B, chains[s, t, :h - k],
                                              hdr.quant_shift, TABLE_MODE, TABLE_BITS,
                                              roots[s >> h, t >> h, c].astype(np.int32), out)
                    assert st == 0
                    planes[s, t, c] = out
        assert sha(planes.astype("<i4")) == str(g[f"planes_k{k}_sha"]), k


def test_corrupt_streams_return_reference_codes(kb):
    import json
    import os
    from paper_1805_06019_b200 import container
    with open(os.path.join(GOLD, "corrupt.json")) as f:
        cases = json.load(f)
    seen = set()
    for case in cases:
        hdr, roots, offs, srv, chains, m = _state(case["name"])
        h, B = hdr.tree_height, hdr.block_size
        wb, hb = hdr.block_grid
        for call in case["calls"]:
            parts = call["call"].split()
            if parts[0] != "decode_plane":
                continue
            s, t, c, k = map(int, parts[1:])
            out = np.empty(roots.shape[3:], np.int32)
            st = kb.decode_plane_core(srv[c], offs[c], wb, hb, m, B, chains[s, t, :h - k], hdr.quant_shift,
                                      TABLE_MODE, TABLE_BITS, roots[s >> h, t >> h, c].astype(np.int32), out)
            want = {None: 0, "corrupt coded pack in SRV payload": 1, "descriptor outside range table": 2}[call["msg"]
                                                                                                         if call["exc"]
                                                                                                         else None]
            assert st == want, call
            seen.add(st)
    assert seen >= {1, 2}


def test_bise_decode_core_vectors(kb):
    import os
    z = np.load(os.path.join(GOLD, "bise_vectors.npz"))
    payload, index, values = z["payload"], z["index"], z["values"]
    from paper_1805_06019_b200.bise import RANGE_TABLE
    starts = np.cumsum([0] + [int(r[1]) for r in index])
    for i, (desc, count, off, nbytes) in enumerate(index[:60]):
        out = np.zeros(int(count), np.uint32)
        r = RANGE_TABLE[int(desc)]
        st = kb.bise_decode_core(payload[off:off + nbytes], int(count), r.mode, r.low_bits, out)
        assert st == 0 and np.array_equal(out, values[starts[i]:starts[i] + count])
    out = np.zeros(5, np.uint32)
    assert kb.bise_decode_core(np.array([243], np.uint8), 5, 1, 0, out) == 1     # pack > 242
