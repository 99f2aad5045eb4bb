"""Reference-side generator of the cfg2 R4 full-field decode golden.

Test infrastructure only (build container; the reference does not travel):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
    PYTHONDONTWRITEBYTECODE=1 python tools/make_cfg2_decode_reference.py STREAM

Runs the LIVE reference decoder on the cfg2 R4 stream (17x17x1024^2, the
bench workload; its sha256 must equal the reference encoder's stream in
tests/golden/cfg2_r4_reference.json).  decode_all (reference
decoder.py:197-210) is decode_image over the S x T grid; as in BASELINE.md
section 3 the images are pooled over a fork multiprocessing.Pool, each worker
calling rlfc.decoder.decode_image (decoder.py:187-194) on its own
DecoderState.  Writes tests/golden/cfg2_r4_decode_reference.json with the
sha256 of the whole (S, T, H, W, 3) uint8 array (C order, the bytes
decode_all returns) and of every image, at stop levels 0 and h.
"""
import hashlib
import json
import multiprocessing as mp
import os
import sys
import time

import numpy as np

from rlfc import decoder

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "..", "tests", "golden", "cfg2_r4_decode_reference.json")

_state = None


def _init(path):
    global _state
    _state = decoder.init(open(path, "rb").read())


def _one(args):
    s, t, k = args
    return s, t, decoder.decode_image(_state, (s, t), stop_level=k).tobytes()


def main(path):
    data = open(path, "rb").read()
    st = decoder.init(data)
    S, T, h = st.header.s_count, st.header.t_count, st.header.tree_height
    res = {"stream_sha256": hashlib.sha256(data).hexdigest(),
           "stream_bytes": len(data), "shape": [S, T, st.header.height,
                                               st.header.width, 3]}
    nproc = os.cpu_count()
    for k in (0, h):
        t0 = time.time()
        with mp.get_context("fork").Pool(nproc, _init, (path,)) as pool:
            imgs = pool.map(_one, [(s, t, k) for s in range(S) for t in range(T)],
                            chunksize=1)
        imgs.sort()
        full = hashlib.sha256()
        per = []
        for s, t, b in imgs:
            full.update(b)
            per.append(hashlib.sha256(b).hexdigest())
        res[f"k{k}"] = {"decode_all_sha256": full.hexdigest(),
                        "image_sha256": per, "seconds": time.time() - t0,
                        "procs": nproc}
        print(k, res[f"k{k}"]["decode_all_sha256"], time.time() - t0, flush=True)
    res["comment"] = ("live reference rlfc 0.1.0 decoder.decode_image pooled "
                      f"over {nproc} forked processes (tools/"
                      "make_cfg2_decode_reference.py)")
    with open(OUT, "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main(sys.argv[1])
