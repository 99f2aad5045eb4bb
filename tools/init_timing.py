"""rl.init wall time on the cfg2 and cfg5 bench streams (process-first and
warm), with the CUDA context created beforehand."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_1805_06019_b200 as rl  # noqa: E402

torch.zeros(1, device="cuda")
torch.cuda.synchronize()
for name, mk in (("cfg2", lambda: bench.make_stream(bench.CFG)[0]), ("cfg5", bench.make_stream_cfg5)):
    data = mk()
    for rep in range(3):
        t0 = time.perf_counter()
        st = rl.init(data)
        torch.cuda.synchronize()
        print(name, "init", rep, round(time.perf_counter() - t0, 4), "s")
        del st
