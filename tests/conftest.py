import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLD = os.path.join(ROOT, "tests", "golden")
STREAMS = os.path.join(GOLD, "streams")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


def golden_names():
    return sorted(f[:-5] for f in os.listdir(STREAMS)
                  if f.endswith(".rlfc") and "_bad_" not in f)


def load_stream(name):
    with open(os.path.join(STREAMS, name + ".rlfc"), "rb") as f:
        return f.read()


_gold_cache = {}


def load_golden(name):
    if name not in _gold_cache:
        z = np.load(os.path.join(GOLD, name + ".npz"))
        g = {k: z[k] for k in z.files}
        g["meta"] = json.loads(str(g["meta"]))
        _gold_cache[name] = g
    return _gold_cache[name]


def sha(a):
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()
