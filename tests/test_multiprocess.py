"""World-size-2 sharding on CPU (gloo): each rank decodes its block-row band
(here with the CPU oracle standing in for its GPU), then gather_field
assembles the full field; it must equal the single-process decode."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT, load_stream


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, name, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle
    from paper_1805_06019_b200 import container, parallel

    class St:
        pass
    data = load_stream(name)
    st = St()
    st.header = container.parse_header(data)
    st.offsets = tuple(container.parse_offsets(data, st.header, c)
                       for c in range(3))
    bands = parallel.balanced_bands(st, world)
    lo, hi = bands[rank]
    B = st.header.block_size
    full, _ = oracle.OracleState(data).decode_all(0, nthreads=1)
    band = torch.from_numpy(np.ascontiguousarray(
        full[:, :, lo * B:min(hi * B, st.header.height)]))
    out = parallel.band_major_to_grid(parallel.gather_field(st, band, bands), st, bands)
    q.put((rank, bool(np.array_equal(out.numpy(), full))))
    dist.destroy_process_group()


@pytest.mark.parametrize("name", ["mid17_r4", "odd_3x5"])
def test_gloo_two_rank_gather(name):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, name, q))
             for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: True, 1: True}


def _gpu_worker(rank, world, port, name, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_1805_06019_b200 as rl
    from paper_1805_06019_b200 import parallel
    torch.cuda.set_device(0)
    st = rl.init(load_stream(name))
    bands = parallel.balanced_bands(st, world)
    band, _ = rl.decode_field(st, 0, rows=bands[rank])          # the real GPU band decode
    full = parallel.band_major_to_grid(parallel.gather_field(st, band.cpu(), bands), st, bands)
    ref, _ = rl.decode_field(st, 0)
    q.put((rank, bool(np.array_equal(full.numpy(), ref.cpu().numpy()))))
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["mid17_r4", "kat8_default"])
def test_two_ranks_gpu_band_decode(name):
    """Two processes on one GPU, each decoding its own block-row band with
    the CUDA path (independent kernels, no cross-rank waiting); the gloo
    band-major gather equals the single-rank decode."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gpu_worker, args=(r, 2, port, name, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: True, 1: True}


@pytest.mark.gpu
def test_bench_two_ranks_one_device():
    """bench.py's N > 1 path end to end (relaunch under torchrun, strong
    scaling over balanced bands, all_gather_into_tensor of the bands, sha256
    parity against the reference golden, max-over-ranks timing) with both
    ranks on cuda:0 over gloo (BENCH_TEST_ONE_DEVICE): the code the driver's
    multi-GPU run executes, minus NCCL."""
    import json
    import subprocess
    import sys
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = dict(os.environ, BENCH_TEST_ONE_DEVICE="1")
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "2", "--warmup",
                        "3", "--no-render", "--no-cpu-baseline"], cwd=ROOT, env=env, capture_output=True,
                       text=True, timeout=900)
    assert p.returncode == 0, p.stderr[-2000:]
    line = json.loads(p.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 2 and line["scaling"] == "strong"
    assert line["parity"]["decode"] == "bit-exact"
    assert len(line["config"]["bands"]) == 2 and line["config"]["bands"][0][0] == 0
    assert line["value"] is not None and "test_hook" in line["config"]
