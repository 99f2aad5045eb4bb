"""RKV/SRV tree construction and record serialisation on the GPU
(producer.encode_gpu, csrc/rlfc_encode.cu) reproduce the reference
encoder's streams byte for byte: every reference-encoded golden stream, the
W >= 256 goldens and the cfg2 R4 bench stream."""
import hashlib
import json
import os

import numpy as np
import pytest

from conftest import GOLD, load_stream
from large_fields import golden

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pr():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1805_06019_b200 import producer
    return producer


def _manifest():
    with open(os.path.join(GOLD, "encoded_manifest.json")) as f:
        return json.load(f)


def _params(d):
    from paper_1805_06019_b200 import encoder
    d = dict(d)
    if "filter" in d:
        d["filter"] = encoder.FilterSpec(kind=d["filter"])
    return encoder.EncodingParams(**d)


@pytest.mark.parametrize("name", sorted(_manifest()))
def test_gpu_encoder_matches_reference_stream(pr, name):
    from paper_1805_06019_b200 import lightfield
    m = _manifest()[name]
    lf = lightfield.synthesize_lightfield(lightfield.SyntheticSpec(**m["spec"]))
    data, _ = pr.encode_gpu(lf, _params(m["params"]))
    assert data == load_stream(name)


@pytest.mark.parametrize("name", sorted(golden()))
def test_gpu_encoder_large(pr, name):
    from paper_1805_06019_b200 import encoder, lightfield
    g = golden()[name]
    lf = lightfield.synthesize_lightfield(lightfield.SyntheticSpec(**g["spec"]))
    data, present = pr.encode_gpu(lf, encoder.EncodingParams(**g["params"]))
    assert hashlib.sha256(data).hexdigest() == g["stream_sha256"]
    assert list(present) == g["present_blocks"]


def test_gpu_encoder_cfg2(pr):
    import time
    from paper_1805_06019_b200 import encoder, lightfield
    with open(os.path.join(GOLD, "cfg2_r4_reference.json")) as f:
        ref = json.load(f)
    lf = lightfield.synthesize_lightfield(lightfield.SyntheticSpec(**ref["spec"]))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    data, present = pr.encode_gpu(lf, encoder.EncodingParams(**ref["params"]))
    dt = time.perf_counter() - t0
    assert hashlib.sha256(data).hexdigest() == ref["stream_sha256"]
    assert list(present) == ref["present_blocks"]
    print(f"cfg2 GPU encode {dt:.2f} s")
