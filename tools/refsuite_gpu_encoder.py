"""rlfc.encoder stand-in for the reference-suite shim's "encoder" route
(tools/refsuite_shim.py): the reference's compress() signature and report,
implemented by paper_1805_06019_b200.encoder.compress with the RKV/SRV trees
and records built on the GPU (producer.encode_gpu).  Test infrastructure."""
from paper_1805_06019_b200.encoder import EncodeReport  # noqa: F401
from paper_1805_06019_b200.encoder import compress as _compress


def compress(lf, params=None):
    return _compress(lf, params, device="cuda")
