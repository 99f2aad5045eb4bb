"""Reference-side generator of tests/golden/cfg2_r4_reference.json.

Runs the live reference (PYTHONPATH=/root/reference/pkg/src) on the cfg2
headline workload: 17x17x1024^2 synthetic field, R4 preset (SURVEY.md
Appendix B).  Takes ~9 minutes and ~14 GB RAM.
"""
import hashlib
import json
import time

from rlfc import encoder
from rlfc.hierarchy import EncodingParams
from rlfc.lightfield import SyntheticSpec, synthesize_lightfield

t0 = time.time()
lf = synthesize_lightfield(SyntheticSpec(17, 17, 1024, 1024, 7))
t1 = time.time()
params = EncodingParams(tree_height=3, block_size=4, quant_shift=4,
                        pixel_threshold=16, block_threshold=1000)
data, rep = encoder.compress(lf, params)
t2 = time.time()
print(json.dumps({
    "rgb_sha256": hashlib.sha256(lf.rgb.tobytes()).hexdigest(),
    "stream_bytes": len(data),
    "stream_sha256": hashlib.sha256(data).hexdigest(),
    "present_blocks": list(rep.present_blocks),
    "synth_s": t1 - t0, "encode_s": t2 - t1}, indent=1))
