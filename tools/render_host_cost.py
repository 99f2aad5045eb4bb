"""Host-side cost of small slab renders and decode_block on the cfg2 R4 stream
(best of three loops of 1000 calls; run old and new package files on one box
to compare)."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import torch, bench, paper_1805_06019_b200 as rl
data, _ = bench.make_stream(bench.CFG)
st = rl.init(data)
h = st.header.tree_height
one = [rl.SlabPose(7.3, 4.6, 512, 512)]
for _ in range(50): rl.render_views(st, one)
torch.cuda.synchronize()
def tm(label, fn, n=1000):
    best = []
    for rep in range(3):
        t0 = time.perf_counter()
        for _ in range(n): fn()
        torch.cuda.synchronize()
        best.append((time.perf_counter()-t0)/n*1e6)
    print(f"{label}: {min(best):.1f} us (min of 3 x {n})")
tm("render_views b1 k0", lambda: rl.render_views(st, one))
tm("render_views b1 kh", lambda: rl.render_views(st, one, stop_level=h))
tm("render_view b1 k0 (host result)", lambda: rl.render_view(st, one[0]))
tm("decode_block", lambda: rl.decode_block(st, (3, 4), (10, 20), 1), n=5000)
tm("decode_image", lambda: rl.decode_image(st, (3, 4)), n=300)
tm("decode_plane", lambda: rl.decode_plane(st, 3, 4, 1), n=300)
