"""Shared helpers for the W >= 256 golden fields (tests/golden/large.json,
made by the live reference with tools/make_goldens_large.py).  The streams
are regenerated here by the native producer and must hash to the reference
encoder's stream sha256 before anything is compared."""
import hashlib
import json
import os

from conftest import GOLD, ROOT

_cache = {}


def golden():
    with open(os.path.join(GOLD, "large.json")) as f:
        return {k: v for k, v in json.load(f).items() if not k.startswith("_")}


def stream(name):
    if name in _cache:
        return _cache[name]
    from paper_1805_06019_b200 import encoder, lightfield
    g = golden()[name]
    path = os.path.join(ROOT, "data", f"golden_{name}_{g['stream_sha256'][:12]}.rlfc")
    if os.path.exists(path):
        with open(path, "rb") as f:
            data = f.read()
    else:
        lf = lightfield.synthesize_lightfield(lightfield.SyntheticSpec(**g["spec"]))
        data, _ = encoder.compress(lf, encoder.EncodingParams(**g["params"]))
        os.makedirs(os.path.dirname(path), exist_ok=True)
        with open(path + f".tmp{os.getpid()}", "wb") as f:
            f.write(data)
        os.replace(path + f".tmp{os.getpid()}", path)
    assert hashlib.sha256(data).hexdigest() == g["stream_sha256"], name
    _cache[name] = data
    return data


def cfg2_stream():
    """The bench's cfg2 R4 stream (17x17x1024^2), produced on demand; its
    sha256 must equal the reference encoder's (cfg2_r4_reference.json)."""
    import sys
    sys.path.insert(0, ROOT)
    import bench
    data, _ = bench.make_stream(bench.CFG)
    with open(os.path.join(GOLD, "cfg2_r4_reference.json")) as f:
        want = json.load(f)["stream_sha256"]
    assert hashlib.sha256(data).hexdigest() == want
    return data
