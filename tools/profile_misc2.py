"""Driver for ncu captures of the kernels added in round 2 beyond the
decode step: the GPU tree construction (k_enc_planes, k_enc_pyramid,
k_enc_srv, k_enc_rec_size, k_enc_records) at cfg2 R4 and the slot-mode
payload pass of a batch-1 render (k_sel_nodes, k_payloads_sel).

    ncu --set full --clock-control none -k regex:'k_enc|k_sel|k_payloads_sel' \\
        -o gpurun_out/misc2 python tools/profile_misc2.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_1805_06019_b200 as rl  # noqa: E402
from paper_1805_06019_b200 import encoder, lightfield, producer  # noqa: E402

spec = lightfield.SyntheticSpec(17, 17, 1024, 1024, 7)
params = encoder.EncodingParams(tree_height=3, block_size=4, quant_shift=4, pixel_threshold=16,
                                block_threshold=1000)
lf = lightfield.synthesize_lightfield(spec)
w = np.ascontiguousarray(producer.pyramid_weights(lf.camera_positions, 3, params.filter))
producer._encode_rows_gpu(lf.rgb, 17, 17, 1024, 1024, 1024, params, w)
del lf
data, _ = bench.make_stream(bench.CFG)
st = rl.init(data)
for _ in range(2):
    rl.render_views(st, [rl.SlabPose(7.3, 4.6, 512, 512)])
torch.cuda.synchronize()
print("ok")
