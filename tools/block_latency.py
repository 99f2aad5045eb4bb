"""Single-block decode latency through the public API (decode_block), as a
host application calls it: 2,000 random picks on the bench stream."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_1805_06019_b200 as rl  # noqa: E402

data, _ = bench.make_stream(bench.CFG)
st = rl.init(data)
hdr = st.header
wb, hb = hdr.block_grid
rng = np.random.default_rng(7)
picks = [(int(rng.integers(0, hdr.s_count)), int(rng.integers(0, hdr.t_count)),
          int(rng.integers(0, wb)), int(rng.integers(0, hb)), int(rng.integers(0, 3)))
         for _ in range(2000)]
for s, t, bx, by, c in picks[:50]:
    rl.decode_block(st, (s, t), (bx, by), c)
t0 = time.perf_counter()
for s, t, bx, by, c in picks:
    rl.decode_block(st, (s, t), (bx, by), c)
dt = (time.perf_counter() - t0) / len(picks)
print(f"decode_block latency {dt * 1e6:.2f} us (mean of {len(picks)})")

# breakdown: the native call alone (no Python argument checks / copy)
from paper_1805_06019_b200 import decoder  # noqa: E402
sc = decoder._block_scratch(st)
ref, mb, stream = sc.args
idle = decoder.BLOCK_SERVER_IDLE_NS
op = sc.out_ptr
t0 = time.perf_counter()
for s, t, bx, by, c in picks:
    sc.fn(ref, mb, s, t, bx, by, c, 0, idle, sc.index_ptr, op, stream)
dt2 = (time.perf_counter() - t0) / len(picks)
print(f"native rlfc_block_server_request alone {dt2 * 1e6:.2f} us")
# the same block over and over (record and roots L2-resident)
s, t, bx, by, c = picks[0]
t0 = time.perf_counter()
for _ in range(len(picks)):
    sc.fn(ref, mb, s, t, bx, by, c, 0, idle, sc.index_ptr, op, stream)
dt3 = (time.perf_counter() - t0) / len(picks)
print(f"native call, one block repeated (L2-warm) {dt3 * 1e6:.2f} us")
# one launch per request (rlfc_decode_block_sync: kernel + polled status)
from paper_1805_06019_b200 import _native  # noqa: E402
import torch  # noqa: E402
L = _native.lib()
host = torch.empty(st.header.block_size ** 2 + 1, dtype=torch.int32).pin_memory()
s2 = torch.cuda.Stream()
t0 = time.perf_counter()
for s, t, bx, by, c in picks:
    L.rlfc_decode_block_sync(ref, s, t, bx, by, c, 0, None, host.data_ptr(), s2.cuda_stream)
dt5 = (time.perf_counter() - t0) / len(picks)
print(f"native rlfc_decode_block_sync (a launch per request) {dt5 * 1e6:.2f} us")
import torch  # noqa: E402
x = torch.zeros(1, device="cuda")
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(len(picks)):
    x.add_(1)
    torch.cuda.synchronize()
dt4 = (time.perf_counter() - t0) / len(picks)
print(f"torch one-kernel launch + synchronize {dt4 * 1e6:.2f} us")

# the Python side of decode_block alone: the native call replaced by a no-op
def _py_cost(label, fn, n=20000):
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    print(f"{label} {(time.perf_counter() - t0) / n * 1e6:.3f} us")


_py_cost("torch.cuda.current_device()", torch.cuda.current_device)
_py_cost("state.device_field()", st.device_field)
_py_cost("decoder._block_scratch(state)", lambda: decoder._block_scratch(st))
real = sc.call_fn
sc.call_fn = lambda p: 0
s, t, bx, by, c = picks[0]
_py_cost("decode_block with a no-op native call", lambda: rl.decode_block(st, (s, t), (bx, by), c))
sc.call_fn = real
