"""Reference-side goldens for W >= 256 fields (test infrastructure only).

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
    PYTHONDONTWRITEBYTECODE=1 python tools/make_goldens_large.py

The LIVE reference (rlfc 0.1.0) synthesizes each light field
(lightfield.py:245-302), encodes it (encoder.compress, encoder.py:23-57),
decodes it (decoder.decode_image pooled over forked processes = decode_all,
decoder.py:187-210) at every stop level, decodes random blocks
(decode_block_progressive, decoder.py:81-106) and renders 512x512 slab views
(render_view, renderer.py:279-305).  Only hashes (and the small block
values) are stored, in tests/golden/large.json: the streams themselves are
regenerated on the test box by the native producer, whose output must hash
to the reference's stream sha256 before anything is compared.
"""
import hashlib
import json
import multiprocessing as mp
import os
import time

import numpy as np

from rlfc import decoder, encoder, renderer
from rlfc.hierarchy import EncodingParams
from rlfc.lightfield import SyntheticSpec, synthesize_lightfield
from rlfc.renderer import SlabPose

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "..", "tests", "golden", "large.json")

R4 = dict(tree_height=3, block_size=4, quant_shift=4, pixel_threshold=16, block_threshold=1000)
CASES = {
    # B = 4 with W >= 256: the staged blend runs >= 4 column chunks per row
    "w256_r4": (dict(s_count=17, t_count=17, width=256, height=256, seed=7), R4),
    "w512_default": (dict(s_count=8, t_count=8, width=512, height=512, seed=7), dict()),
    "w512_b8": (dict(s_count=8, t_count=8, width=512, height=512, seed=3), dict(block_size=8, tree_height=3)),
    "w512_b16": (dict(s_count=8, t_count=8, width=512, height=512, seed=5),
                 dict(block_size=16, tree_height=3, quant_shift=2, pixel_threshold=4, block_threshold=60)),
    # B = 4 with quant_shift > 4: residuals exceed int16, the blend's 32-bit path
    "w256_b4_s5": (dict(s_count=9, t_count=9, width=256, height=256, seed=17),
                   dict(tree_height=3, block_size=4, quant_shift=5, pixel_threshold=24, block_threshold=2000)),
    "w256_b4_s6_dense": (dict(s_count=9, t_count=9, width=256, height=256, seed=19),
                         dict(tree_height=3, block_size=4, quant_shift=6, pixel_threshold=2, block_threshold=40)),
}
_st = None


def _init(data):
    global _st
    _st = decoder.init(data)


def _img(args):
    s, t, k = args
    return s, t, decoder.decode_image(_st, (s, t), stop_level=k).tobytes()


def sha(b):
    return hashlib.sha256(b).hexdigest()


def main():
    import sys
    only = sys.argv[1].split(",") if len(sys.argv) > 1 else None   # add / redo these, keep the rest
    res = {}
    if only and os.path.exists(OUT):
        with open(OUT) as f:
            res = json.load(f)
    for name, (spec, params) in CASES.items():
        if only and name not in only:
            continue
        t0 = time.time()
        lf = synthesize_lightfield(SyntheticSpec(**spec))
        data, rep = encoder.compress(lf, EncodingParams(**params))
        st = decoder.init(data)
        hdr = st.header
        S, T, h, B = hdr.s_count, hdr.t_count, hdr.tree_height, hdr.block_size
        wb, hb = hdr.block_grid
        entry = {"spec": spec, "params": params, "stream_sha256": sha(data), "stream_bytes": len(data),
                 "present_blocks": list(rep.present_blocks), "S": S, "T": T, "W": hdr.width,
                 "H": hdr.height, "B": B, "h": h}
        with mp.get_context("fork").Pool(os.cpu_count(), _init, (data,)) as pool:
            for k in range(h + 1):
                imgs = sorted(pool.map(_img, [(s, t, k) for s in range(S) for t in range(T)]))
                hsh = hashlib.sha256()
                for _, _, b in imgs:
                    hsh.update(b)
                entry[f"all_k{k}_sha"] = hsh.hexdigest()
        rng = np.random.default_rng(13)
        blocks = []
        for _ in range(40):
            s, t = int(rng.integers(0, S)), int(rng.integers(0, T))
            bx, by = int(rng.integers(0, wb)), int(rng.integers(0, hb))
            c, k = int(rng.integers(0, 3)), int(rng.integers(0, h + 1))
            v = decoder.decode_block_progressive(st, (s, t), (bx, by), c, k)
            blocks.append([s, t, bx, by, c, k, v.astype(np.int64).ravel().tolist()])
        entry["blocks"] = blocks
        renders = []
        prng = np.random.default_rng(29)
        for i, (focal, k) in enumerate([(None, 0), (0.9, 0), (1.12, 0), (None, min(2, h)), (None, 0)]):
            s = float(prng.uniform(0, S - 1))
            t = float(prng.uniform(0, T - 1))
            pose = SlabPose(s, t, 512, 512, focal_z=focal)
            img = renderer.render_view(st, pose, stop_level=k)
            renders.append({"s": s, "t": t, "focal_z": focal, "k": k, "sha256": sha(img.tobytes())})
        entry["renders"] = renders
        entry["seconds"] = time.time() - t0
        res[name] = entry
        print(name, len(data), entry["all_k0_sha"][:16], f"{entry['seconds']:.0f}s", flush=True)
    res["_comment"] = ("live reference rlfc 0.1.0: synthesize_lightfield + encoder.compress + "
                       "decode_image pooled over forked processes + decode_block_progressive + "
                       "render_view (tools/make_goldens_large.py)")
    with open(OUT, "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
