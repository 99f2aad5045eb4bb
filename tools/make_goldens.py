"""Generate the golden fixtures under tests/golden/ from the LIVE reference.

Test infrastructure only.  Run in the build container, where the reference
package is importable read-only:

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
    PYTHONDONTWRITEBYTECODE=1 python tools/make_goldens.py

Every stream is produced by the reference encoder (`rlfc.encoder.compress`,
reference pkg/src/rlfc/encoder.py:23-57) or, for the hand-crafted descriptor
sweep, by the reference serializer (`rlfc.container.serialize`,
container.py:269-339) over a synthetic SRV tree.  Every expected output is the
reference decoder / renderer run on that stream (decoder.py:81-210,
renderer.py:147-305).  The fixtures travel to the GPU box; the reference does
not, so nothing at test time imports it.
"""

import hashlib
import json
import os
import sys

import numpy as np

from rlfc import bise, container, decoder, encoder, renderer
from rlfc.errors import FormatError
from rlfc.hierarchy import (EncodingParams, FilterSpec, SrvChannelNode,
                            SrvLevel, SrvTree)
from rlfc.lightfield import (PlaneGeometry, SyntheticSpec,
                             synthesize_lightfield)
from rlfc.renderer import CameraPose, SlabPose

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = os.path.join(HERE, "..", "tests", "golden")
STREAMS = os.path.join(GOLD, "streams")


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def P(**kw):
    return EncodingParams(**kw)


# name -> (SyntheticSpec kwargs, EncodingParams kwargs)
ENCODED = {
    # reference KAT stream: test_encoder.py:26-34 (194,323 B)
    "kat8_default": (dict(), dict()),
    "kat8_lossless": (dict(), dict(pixel_threshold=0, block_threshold=0,
                                   quant_shift=0, root_codec="raw")),
    # cfg1 (BASELINE.json configs[0]): 8x8x64^2, B=4, h=2
    "cfg1_h2": (dict(), dict(tree_height=2, quant_shift=4, pixel_threshold=8,
                             block_threshold=600, root_codec="raw")),
    "cfg1_h3_r4": (dict(), dict(tree_height=3, quant_shift=4,
                                pixel_threshold=16, block_threshold=1000)),
    "b2_h1": (dict(s_count=4, t_count=4, width=32, height=32, seed=11),
              dict(block_size=2, tree_height=1, root_codec="raw")),
    "b8_h2": (dict(s_count=4, t_count=4, width=32, height=32, seed=11),
              dict(block_size=8, tree_height=2, root_codec="raw")),
    "b16_h4": (dict(), dict(block_size=16, tree_height=4, quant_shift=1,
                            pixel_threshold=2, block_threshold=20,
                            root_codec="raw")),
    "odd_3x5": (dict(s_count=3, t_count=5, width=30, height=22, seed=3),
                dict(tree_height=2, quant_shift=1, pixel_threshold=2,
                     block_threshold=10, root_codec="raw")),
    "uniform_5x3": (dict(s_count=5, t_count=3, width=20, height=36, seed=5),
                    dict(tree_height=2, quant_shift=0, pixel_threshold=1,
                         block_threshold=1, root_codec="raw",
                         filter=FilterSpec(kind="uniform"))),
    # cfg2 shape (17x17 grid, M=395) at reduced resolution, R4 preset
    "mid17_r4": (dict(s_count=17, t_count=17, width=64, height=64),
                 dict(tree_height=3, quant_shift=4, pixel_threshold=16,
                      block_threshold=1000)),
    # cfg2 shape, dense R6-like preset
    "mid17_dense": (dict(s_count=17, t_count=17, width=32, height=32),
                    dict(tree_height=3, quant_shift=1, pixel_threshold=1,
                         block_threshold=1, root_codec="raw")),
    # R1 preset shape: h=5, B=16, no residual blocks at all
    "r1_empty": (dict(s_count=17, t_count=17, width=48, height=48),
                 dict(tree_height=5, block_size=16, quant_shift=6,
                      pixel_threshold=64, block_threshold=1000000,
                      root_codec="raw")),
    # 32x32 grid at tiny resolution (cfg5 node count M=1344)
    "grid32": (dict(s_count=32, t_count=32, width=16, height=16),
               dict(tree_height=3, quant_shift=2, pixel_threshold=2,
                    block_threshold=30, root_codec="raw")),
}


def slab_poses(S, T, W, H):
    poses = [SlabPose(float(min(3, S - 1)), float(min(4, T - 1)), W, H),
             SlabPose(min(3.5, S - 1.0), min(4.25, T - 1.0), 32, 32),
             SlabPose(min(2.3, S - 1.0), min(6.9, T - 1.0), 24, 24,
                      focal_z=1.12),
             SlabPose(-0.5, min(3.0, T - 1.0), 16, 16),
             SlabPose(S - 1.001, 0.001, 24, 24, focal_z=0.9),
             SlabPose(S + 0.7, T - 0.3, 20, 12)]
    rng = np.random.default_rng(31)
    for _ in range(3):
        poses.append(SlabPose(float(rng.uniform(0, S - 1)),
                              float(rng.uniform(0, T - 1)), 48, 40))
    return poses


def pose_json(p):
    if isinstance(p, SlabPose):
        return {"kind": "slab", "s": p.s, "t": p.t, "width": p.width,
                "height": p.height, "focal_z": p.focal_z}
    return {"kind": "camera", "eye": list(p.eye), "look": list(p.look),
            "fov_deg": p.fov_deg, "width": p.width, "height": p.height}


def golden_for_stream(name, data, enc_report=None, params=None,
                      render=True, pinhole=True, full_rgb=False):
    with open(os.path.join(STREAMS, name + ".rlfc"), "wb") as f:
        f.write(data)
    st = decoder.init(data)
    hdr = st.header
    S, T, W, H = hdr.s_count, hdr.t_count, hdr.width, hdr.height
    h, B = hdr.tree_height, hdr.block_size
    wb, hb = hdr.block_grid
    out = {}
    meta = {
        "name": name, "bytes": len(data),
        "sha256": hashlib.sha256(data).hexdigest(),
        "S": S, "T": T, "W": W, "H": H, "B": B, "h": h,
        "shift": hdr.quant_shift, "codec": hdr.root_codec_id,
        "m_nodes": st.m_nodes, "sections": [list(s) for s in
                                            hdr.section_lengths],
    }
    if enc_report is not None:
        meta["present_blocks"] = list(enc_report.present_blocks)
    if params is not None:
        meta["params"] = {
            "tree_height": params.tree_height,
            "block_size": params.block_size,
            "pixel_threshold": params.pixel_threshold,
            "block_threshold": params.block_threshold,
            "quant_shift": params.quant_shift,
            "filter_kind": params.filter.kind,
            "sigma": params.filter.sigma,
            "root_codec": params.root_codec}
    out["chains"] = st.chains.astype(np.int64)
    out["root_planes_sha"] = np.array(sha(st.root_planes.astype(np.int32)))
    for k in range(h + 1):
        rgb = decoder.decode_all(st, stop_level=k).rgb
        out[f"all_k{k}_sha"] = np.array(sha(rgb))
        if full_rgb and k == 0:
            out["rgb_k0"] = rgb
        planes = np.stack([np.stack([np.stack(
            [decoder.decode_plane(st, s, t, c, k) for c in range(3)])
            for t in range(T)]) for s in range(S)]).astype("<i4")
        out[f"planes_k{k}_sha"] = np.array(sha(planes))
    rng = np.random.default_rng(20)
    nreq = 120
    req = np.zeros((nreq, 6), dtype=np.int32)
    vals = np.zeros((nreq, B, B), dtype=np.int32)
    for i in range(nreq):
        s, t = int(rng.integers(0, S)), int(rng.integers(0, T))
        bx, by = int(rng.integers(0, wb)), int(rng.integers(0, hb))
        c, k = int(rng.integers(0, 3)), int(rng.integers(0, h + 1))
        req[i] = (s, t, bx, by, c, k)
        vals[i] = decoder.decode_block_progressive(st, (s, t), (bx, by), c, k)
    out["blocks_req"] = req
    out["blocks_val"] = vals
    poses = []
    if render:
        for p in slab_poses(S, T, W, H):
            for k in sorted({0, min(2, h)}):
                bg = (9, 8, 7) if p.focal_z is not None else (0, 0, 0)
                img = renderer.render_view(st, p, stop_level=k,
                                           background=bg)
                out[f"render_{len(poses)}"] = img
                poses.append({"pose": pose_json(p), "k": k,
                              "background": list(bg)})
        # refocus so far that rays spill past the extent (background path)
        p = SlabPose(0.0, 0.0, 16, 16, focal_z=0.5)
        out[f"render_{len(poses)}"] = renderer.render_view(
            st, p, background=(9, 8, 7))
        poses.append({"pose": pose_json(p), "k": 0, "background": [9, 8, 7]})
        # non-default geometry
        geo = PlaneGeometry(0.0, 1.6, (-2.0, -1.0, S + 1.0, T + 0.25))
        p = SlabPose(S * 0.37, T * 0.61, 28, 20, focal_z=1.3)
        out[f"render_{len(poses)}"] = renderer.render_view(st, p,
                                                           geometry=geo)
        poses.append({"pose": pose_json(p), "k": 0, "background": [0, 0, 0],
                      "geometry": [geo.camera_plane_z, geo.image_plane_z,
                                   list(geo.image_plane_extent)]})
    if pinhole:
        cams = [CameraPose(eye=(S / 2 - 0.5, T / 2 - 0.5, -2.0),
                           look=(0.0, 0.0, 1.0), fov_deg=50.0, width=24,
                           height=24),
                CameraPose(eye=(1.2, 0.7, -1.5), look=(0.1, 0.05, 1.0),
                           fov_deg=35.0, width=20, height=16),
                CameraPose(eye=(S * 0.5, T * 0.4, 3.0), look=(0.05, -0.1, -1.0),
                           fov_deg=70.0, width=16, height=16)]
        for p in cams:
            for k in sorted({0, min(2, h)}):
                img = renderer.render_view(st, p, stop_level=k)
                out[f"render_{len(poses)}"] = img
                poses.append({"pose": pose_json(p), "k": k,
                              "background": [0, 0, 0]})
    meta["renders"] = poses
    out["meta"] = np.array(json.dumps(meta))
    np.savez_compressed(os.path.join(GOLD, name + ".npz"), **out)
    print(f"{name}: {len(data)} B, M={st.m_nodes}, {len(poses)} renders",
          flush=True)
    return st


def crafted_alldesc(name, S, T, W, Hh, h, B, shift, seed, codec="raw"):
    """Hand-crafted stream: every descriptor 0..29, full-range roots.

    Uses the reference serializer (container.py:269-339) on a synthetic SRV
    tree, so the bytes are exactly what the format defines.
    """
    rng = np.random.default_rng(seed)
    wp = -(-W // B) * B
    hp = -(-Hh // B) * B
    wb, hb = wp // B, hp // B
    rsx, rsy = container.level_dims(S, T, h)
    roots = np.zeros((rsx, rsy, 3, hp, wp), dtype=np.int64)
    roots[:, :, 0] = rng.integers(0, 65536, size=(rsx, rsy, hp, wp))
    roots[:, :, 1:] = rng.integers(-256, 65280, size=(rsx, rsy, 2, hp, wp))
    # mostly-small roots so the clamp is not always saturated
    small = rng.random(size=roots.shape) < 0.7
    roots = np.where(small, rng.integers(-200, 300, size=roots.shape), roots)
    roots[:, :, 0] = np.clip(roots[:, :, 0], 0, 65535)
    roots[:, :, 1:] = np.clip(roots[:, :, 1:], -256, 65279)
    levels = []
    desc_cycle = 0
    for l in range(h):
        sx, sy = container.level_dims(S, T, l)
        nodes = []
        for x in range(sx):
            col = []
            for y in range(sy):
                cell = []
                for c in range(3):
                    present = rng.random((hb, wb)) < 0.6
                    ridx = np.zeros((hb, wb), dtype=np.uint8)
                    z = np.zeros((hb, wb, B * B), dtype=np.uint16)
                    for by in range(hb):
                        for bx in range(wb):
                            if not present[by, bx]:
                                continue
                            d = desc_cycle % 30
                            desc_cycle += 1
                            n = bise.RANGE_CARDINALITIES[d]
                            vals = rng.integers(0, n, size=B * B)
                            if rng.random() < 0.5:
                                vals[rng.integers(0, B * B)] = n - 1
                            z[by, bx] = vals
                            ridx[by, bx] = d
                    cell.append(SrvChannelNode(present, ridx, z))
                col.append(cell)
            nodes.append(col)
        levels.append(SrvLevel(nodes))
    params = EncodingParams(tree_height=h, block_size=B, quant_shift=shift,
                            root_codec=codec)
    data = container.serialize(roots, SrvTree(levels), params, S, T, W, Hh)
    return data


def corrupt_variants(base_name, data):
    """Byte-patched streams and the reference's exact error behaviour."""
    st = decoder.init(data)
    hdr = st.header
    cases = []
    # find present nodes by mode in channel 0/1/2 records
    found = {}
    wb, hb = hdr.block_grid
    for c in range(3):
        for blk in range(wb * hb):
            for ni in range(st.m_nodes):
                got = container.locate_block(data, hdr, c, blk, ni)
                if got is None:
                    continue
                start, end, desc = got
                mode = int(bise.TABLE_MODE[desc])
                key = "desc" if "desc" not in found else (
                    "trit" if mode == 1 else "quint" if mode == 2 else None)
                if key is None or key in found:
                    continue
                found[key] = (c, blk, ni, start, end, desc)
            if len(found) == 3:
                break
        if len(found) == 3:
            break
    for kind, (c, blk, ni, start, end, desc) in found.items():
        bad = bytearray(data)
        if kind == "desc":
            bad[start - 1] = 99
        elif kind == "trit":
            bad[start] = 250            # first pack byte > 242
        else:
            bad[start] = (bad[start] & 0x80) | 126   # 7-bit pack > 124
        bad = bytes(bad)
        name = f"{base_name}_bad_{kind}"
        with open(os.path.join(STREAMS, name + ".rlfc"), "wb") as f:
            f.write(bad)
        bst = decoder.init(bad)
        bx, by = blk % wb, blk // wb
        # which images have this node in their chain
        imgs = [(s, t) for s in range(hdr.s_count) for t in range(hdr.t_count)
                if ni in set(int(v) for v in bst.chains[s, t])]
        s, t = imgs[0]
        calls = []

        def rec(label, fn):
            try:
                fn()
                calls.append({"call": label, "exc": None, "msg": None})
            except FormatError as exc:
                calls.append({"call": label, "exc": type(exc).__name__,
                              "msg": str(exc)})
        rec(f"decode_block {s} {t} {bx} {by} {c} 0", lambda: decoder.decode_block(
            bst, (s, t), (bx, by), c))
        rec(f"decode_block {s} {t} {bx} {by} {c} {hdr.tree_height}",
            lambda: decoder.decode_block_progressive(
                bst, (s, t), (bx, by), c, hdr.tree_height))
        rec(f"decode_plane {s} {t} {c} 0",
            lambda: decoder.decode_plane(bst, s, t, c))
        rec(f"decode_image {s} {t} 0",
            lambda: decoder.decode_image(bst, (s, t)))
        rec("decode_all 0", lambda: decoder.decode_all(bst))
        rec(f"decode_all {hdr.tree_height}",
            lambda: decoder.decode_all(bst, hdr.tree_height))
        cases.append({"name": name, "kind": kind, "channel": c, "blk": blk,
                      "node": ni, "calls": calls})
        print(f"{name}: {[(x['call'], x['exc']) for x in calls]}",
              flush=True)
    return cases


def bise_vectors():
    """Random payloads for every descriptor and several counts."""
    rng = np.random.default_rng(4)
    recs = []
    blobs = []
    for d, e in enumerate(bise.RANGE_TABLE):
        for n in (1, 2, 3, 4, 5, 7, 15, 16, 64, 256):
            vals = rng.integers(0, e.cardinality, size=n).astype(np.uint16)
            data = bise.bise_encode(vals, e)
            recs.append((d, n, len(b"".join(blobs)), len(data)))
            blobs.append(data)
            recs[-1] = recs[-1] + (vals.tolist(),)
    payload = np.frombuffer(b"".join(blobs), dtype=np.uint8)
    index = np.array([r[:4] for r in recs], dtype=np.int64)
    values = np.concatenate([np.asarray(r[4], dtype=np.uint16) for r in recs])
    np.savez_compressed(os.path.join(GOLD, "bise_vectors.npz"),
                        payload=payload, index=index, values=values,
                        table_mode=bise.TABLE_MODE, table_bits=bise.TABLE_BITS,
                        kat=np.frombuffer(bise.bise_encode(
                            np.array([5, 0, 3], np.uint16),
                            bise.RANGE_TABLE[4]), np.uint8))
    print("bise vectors:", len(recs))


def synth_hashes():
    out = {}
    for spec in [SyntheticSpec(), SyntheticSpec(4, 4, 32, 32, 11),
                 SyntheticSpec(17, 17, 64, 64, 7), SyntheticSpec(3, 5, 30, 22, 3),
                 SyntheticSpec(17, 17, 128, 128, 7)]:
        lf = synthesize_lightfield(spec)
        out[f"{spec.s_count}x{spec.t_count}x{spec.width}x{spec.height}"
            f"s{spec.seed}"] = sha(lf.rgb)
    with open(os.path.join(GOLD, "synth_sha256.json"), "w") as f:
        json.dump(out, f, indent=1)


def main():
    os.makedirs(STREAMS, exist_ok=True)
    only = set(sys.argv[1:])
    manifest = {}
    if not only or "bise" in only:
        bise_vectors()
    if not only or "synth" in only:
        synth_hashes()
    for name, (spec_kw, par_kw) in ENCODED.items():
        if only and name not in only:
            continue
        lf = synthesize_lightfield(SyntheticSpec(**spec_kw))
        params = P(**par_kw)
        data, rep = encoder.compress(lf, params)
        big = lf.s_count * lf.t_count * lf.width * lf.height > 400_000
        golden_for_stream(name, data, rep, params,
                          render=True, pinhole=not big,
                          full_rgb=name in ("kat8_default", "odd_3x5"))
        manifest[name] = {"spec": spec_kw, "params": {
            k: (v.kind if isinstance(v, FilterSpec) else v)
            for k, v in par_kw.items()}}
    crafted = {"alldesc_b4": (3, 3, 20, 16, 2, 4, 3, 1),
               "alldesc_b8_s0": (2, 3, 24, 16, 1, 8, 0, 2),
               "alldesc_b2_s8": (5, 2, 6, 10, 2, 2, 8, 3),
               "alldesc_b16": (2, 2, 16, 32, 1, 16, 5, 4)}
    for name, args in crafted.items():
        if only and name not in only:
            continue
        data = crafted_alldesc(name, *args)
        golden_for_stream(name, data, render=True, pinhole=False)
    if not only or "corrupt" in only:
        with open(os.path.join(STREAMS, "kat8_default.rlfc"), "rb") as f:
            base = f.read()
        cases = corrupt_variants("kat8_default", base)
        with open(os.path.join(GOLD, "corrupt.json"), "w") as f:
            json.dump(cases, f, indent=1)
    if manifest:
        path = os.path.join(GOLD, "encoded_manifest.json")
        old = {}
        if os.path.exists(path):
            with open(path) as f:
                old = json.load(f)
        old.update(manifest)
        with open(path, "w") as f:
            json.dump(old, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
