"""Benchmark: full light-field decode (and batched 512x512 rendering) on B200.

Headline workload (BASELINE.json configs[1]): the synthetic
17x17-view 1024x1024 light field, R4 preset (h=3, B=4, s=4, Tp=16, Tb=1000;
1.85 bpp), produced on the box by the native producer (byte-identical to the
reference encoder, tests/test_producer.py).  One step = one full-field decode
of all 289 views (303 Mpix) from the compressed stream resident in HBM to
RGB8 in HBM, by the staged sm_100a decode (record index, payload decode,
TMA-fed blend: four kernel launches per step; --kernel fused runs the single
tiled kernel instead).  Rank 0 prints ONE JSON line.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

N > 1 runs under torchrun, one process per GPU (NCCL for barriers only):
weak scaling, every rank decodes its own light field (independent objects);
--scaling strong instead partitions one field's block rows across ranks,
balanced by compressed bytes.  There is no collective on the data path.
"""

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CFG = dict(S=17, T=17, W=1024, H=1024, seed=7, h=3, B=4, shift=4, tp=16,
           tb=1000, codec="png")
PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
L2_BYTES = 126 * 1024 * 1024


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def make_stream(cfg, cache_dir=os.path.join(ROOT, "data")):
    """Produce (or reuse) the benchmark stream: RKV/SRV trees built on the
    GPU (producer.encode_gpu), byte-identical to the reference encoder."""
    import hashlib
    from paper_1805_06019_b200 import encoder, lightfield
    key = hashlib.sha1(json.dumps(cfg, sort_keys=True).encode()).hexdigest()[:12]
    path = os.path.join(cache_dir, f"bench_{key}.rlfc")
    if os.path.exists(path):
        with open(path, "rb") as f:
            return f.read(), path
    t0 = time.time()
    lf = lightfield.synthesize_lightfield(lightfield.SyntheticSpec(
        cfg["S"], cfg["T"], cfg["W"], cfg["H"], cfg["seed"]))
    params = encoder.EncodingParams(
        tree_height=cfg["h"], block_size=cfg["B"], quant_shift=cfg["shift"],
        pixel_threshold=cfg["tp"], block_threshold=cfg["tb"],
        root_codec=cfg["codec"])
    import torch
    dev = "cuda" if torch.cuda.is_available() else None
    data, rep = encoder.compress(lf, params, device=dev)
    log(f"produced stream {len(data)} B ({rep.bpp_total:.3f} bpp) in "
        f"{time.time() - t0:.1f}s; present per level {rep.present_blocks}")
    os.makedirs(cache_dir, exist_ok=True)
    tmp = path + f".tmp{os.getpid()}"
    with open(tmp, "wb") as f:
        f.write(data)
    os.replace(tmp, path)
    return data, path


def stream_stats(state):
    hdr = state.header
    S, T, W, H = hdr.s_count, hdr.t_count, hdr.width, hdr.height
    wp, hp = hdr.padded_dims
    wb, hb = hdr.block_grid
    from paper_1805_06019_b200 import container
    rsx, rsy = container.level_dims(S, T, hdr.tree_height)
    comp = sum(sec[1] + sec[2] for sec in hdr.section_lengths)
    roots = 3 * rsx * rsy * hp * wp * 2
    out = S * T * W * H * 3
    present = 0
    for c in range(3):
        srv = state.srv[c]
        offs = state.offsets[c].astype(np.int64)
        nbm = (state.m_nodes + 7) >> 3
        bm = srv[(offs[:, None] + np.arange(nbm)[None, :])]
        present += int(np.unpackbits(bm, axis=1, bitorder="little")
                       [:, :state.m_nodes].sum())
    return dict(pixels=S * T * W * H, comp_bytes=comp, root_bytes=roots,
                out_bytes=out, alg_bytes=comp + roots + out,
                bpp=8.0 * len(state.data) / (S * T * W * H),
                present=present, present_frac=present / (state.m_nodes * wb * hb * 3))


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            self.proc.wait()
            self.thread.join(timeout=2)

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown",
                 "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                mx = float(r[1])
                for n, v in zip(names, r[4:8]):
                    if v.lower().startswith("active"):
                        reasons.add(n)
            except (ValueError, IndexError):
                continue
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


NCU_SUMMARY = {"fused": "profiles/r1_decode_ncu_summary.json",
               "staged": "profiles/r2_staged_ncu_summary.json"}
KERNELS = {"dir": ["k_seg_dir"],
           "fused": ["k_decode_field_tiled"],
           "staged": ["k_payloads", "k_blend"],
           "simple": ["k_decode_field_simple"]}


def ncu_traffic(kernel_kind):
    """DRAM bytes per decode step (all of the step's kernels) from the
    committed ncu capture of the same path, or None."""
    rel = NCU_SUMMARY.get(kernel_kind)
    path = os.path.join(ROOT, rel) if rel else None
    if not path or not os.path.exists(path):
        return None, None
    try:
        with open(path) as f:
            return int(json.load(f)["dram_bytes_total"]), rel
    except (OSError, KeyError, ValueError):
        return None, None


def peaks():
    try:
        with open(PEAKS) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback"


# --- CPU baseline / reference arm -------------------------------------------------

def cpu_decode(data, steps, warmup, cfg_name, want_sha=False):
    """Oracle port (C restatement of the reference decode path), all host
    threads, full field per step."""
    from oracle import oracle
    oracle.build()
    orc = oracle.OracleState(data)
    nth = oracle.lib().orc_nproc()
    times = []
    for i in range(warmup + steps):
        t0 = time.perf_counter()
        out, st = orc.decode_all(0, nthreads=nth)
        dt = time.perf_counter() - t0
        assert st == 0
        if i >= warmup:
            times.append(dt)
    px = orc.S * orc.T * orc.W * orc.H
    if want_sha:
        import hashlib
        return px / statistics.mean(times) / 1e9, nth, times, hashlib.sha256(out.tobytes()).hexdigest()
    return px / statistics.mean(times) / 1e9, nth, times


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    data, _ = make_stream(CFG)
    val, nth, times = cpu_decode(data, args.steps, args.warmup, "cfg2")
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": "Gpix/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000 * statistics.mean(times),
        "higher_is_better": True, "scaling": args.scaling or ("strong" if args.gpus > 1 else "weak"),
        "vs_baseline": None, "dtype": "int32", "data": "synthetic",
        "config": dict(workload_config(), bpp=round(8.0 * len(data) / (289 * 1024 * 1024), 4),
                       present_frac=0.06449, kernel="oracle C port (reference decode_all order)",
                       bands=[[0, 256]]),
        "cpu_baseline": {"value": val, "unit": "Gpix/s", "cores": nth,
                         "kind": "port",
                         "sample": "full 17x17x1024^2 field per step"},
        "e2e": {"value": val, "unit": "Gpix/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


METRIC = "decoded Gpixels/s (full light-field decode, cfg2 R4)"


def workload_config():
    return {"workload": "full-field decode, 17x17 views x 1024x1024 RGB, "
                        "R4 (h=3 B=4 s=4 Tp=16 Tb=1000)",
            "preset": "R4", "views": 289, "width": 1024, "height": 1024,
            "block": 4, "tree_height": 3,
            "l2": "working set > L2 (0.9 GB output per step), no flush"}


# --- GPU arm -----------------------------------------------------------------------

REF_DECODE = os.path.join(ROOT, "tests", "golden", "cfg2_r4_decode_reference.json")


def relaunch(args):
    """--gpus N without a launcher: re-run this script under torchrun, one
    process per GPU (rank 0 prints the line)."""
    import socket
    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def sha_host(t):
    import hashlib
    return hashlib.sha256(t.cpu().numpy().tobytes()).hexdigest()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--scaling", default=None, choices=["weak", "strong"],
                    help="N > 1: strong (default; cfg3, one cfg2 field split "
                         "into block-row bands) or weak (a field per rank)")
    ap.add_argument("--kernel", default="auto", choices=["auto", "staged", "dir", "fused", "simple"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-render", action="store_true")
    ap.add_argument("--config", default="cfg2", choices=["cfg2", "cfg5"])
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference_arm(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch(args)
    if args.config == "cfg5":
        return run_cfg5(args)
    for k in os.environ:
        if k.startswith("RLFC_"):
            raise SystemExit(f"refusing to benchmark with {k} set")

    import torch
    import torch.distributed as dist
    import paper_1805_06019_b200 as rl
    from paper_1805_06019_b200 import decoder, parallel

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # test hook for the N > 1 code path on a one-GPU box: every rank on
    # cuda:0, gloo instead of NCCL (NCCL refuses two ranks on one device);
    # its numbers are not a scaling measurement
    one_dev = os.environ.get("BENCH_TEST_ONE_DEVICE") == "1"
    if one_dev:
        local = 0
    torch.cuda.set_device(local)
    scaling = args.scaling or ("strong" if world > 1 else "weak")
    if world > 1:
        if one_dev:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def barrier():
        if world > 1:
            dist.barrier()

    data, _ = make_stream(CFG) if rank == 0 or world == 1 else (None, None)
    if world > 1:
        obj = [data]
        dist.broadcast_object_list(obj, src=0)
        data = obj[0]
    state = rl.init(data)
    hdr = state.header
    st = stream_stats(state)
    hb = hdr.block_grid[1]
    B = hdr.block_size
    if scaling == "strong" and world > 1:
        bands = parallel.balanced_bands(state, world)
    else:
        bands = [(0, hb)] * world
    band = bands[rank]
    rows_px = min(band[1] * B, hdr.height) - band[0] * B
    px_rank = hdr.s_count * hdr.t_count * hdr.width * rows_px
    out = torch.empty((hdr.s_count, hdr.t_count, rows_px, hdr.width, 3),
                      dtype=torch.uint8, device="cuda")
    stream = torch.cuda.current_stream()
    kern = "staged" if args.kernel == "auto" else args.kernel
    # stream-invariant record index (built once per workspace): timed here
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    prepared = state.device_field().staged_workspace(stream.cuda_stream) if kern == "staged" else None
    torch.cuda.synchronize()
    index_ms = (time.perf_counter() - t0) * 1e3

    def step():
        decoder.decode_field(state, 0, rows=band, out=out, kernel=kern, check=False)

    # correctness gate before timing: status word must be clean
    decoder.decode_field(state, 0, rows=band, out=out, kernel=kern, check=True)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        # soak: the same step back to back for >= 1 s so nvidia-smi (100 ms
        # period) samples the clocks under this load; the timed region
        # follows immediately, still inside the sampling window
        t_soak = time.perf_counter()
        while time.perf_counter() - t_soak < 1.0:
            for _ in range(4):
                step()
            torch.cuda.synchronize()
        barrier()
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        torch.cuda.synchronize()
        barrier()
    ms = ev0.elapsed_time(ev1) / args.steps
    per_rank = [ms]
    if world > 1:
        per_rank = [None] * world
        dist.all_gather_object(per_rank, ms)
    ms_max = max(per_rank)
    total_px = px_rank * world if scaling == "weak" else \
        hdr.s_count * hdr.t_count * hdr.width * hdr.height
    value = total_px / (ms_max * 1e-3) / 1e9

    # parity: the decoded field against the live reference's decode_all
    # sha256 (and the oracle's, when the CPU leg runs); strong scaling
    # assembles the bands on rank 0 with one all_gather_into_tensor
    parity = parity_check(state, out, bands, scaling, world, rank, parallel)

    # roofline of the step on this rank: algorithmic bytes (SURVEY 8d
    # formula) plus the per-step reads of the prepared record index
    frac_rows = rows_px / hdr.height
    idx_bytes = (8 * st["present"] + 4 * 3 * hdr.block_grid[0] * hb +
                 2 * 4 * ((state.m_nodes + 31) // 32 + 2) * 3 * hdr.block_grid[0] * hb)
    alg = (st["comp_bytes"] + st["root_bytes"] + st["out_bytes"] + idx_bytes) * frac_rows
    achieved = alg / (ms * 1e-3) / 1e9
    peak, peak_kind = peaks()

    e2e = e2e_measure(state, band, args, rl)
    render = None if args.no_render else render_measure(state, args, rl, world, rank)
    random_access = random_access_measure(state, rl)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        val, nth, times, orc_sha = cpu_decode(data, 2, 1, "cfg2", want_sha=True)
        cpu = {"value": val, "unit": "Gpix/s", "cores": nth, "kind": "port",
               "sample": "full 17x17x1024^2 R4 field, oracle C port, "
                         f"{nth} threads, mean of {len(times)} steps"}
        parity["oracle_sha256"] = orc_sha
        if parity.get("sha256") and orc_sha != parity["sha256"]:
            parity["decode"] = "MISMATCH (oracle)"

    traffic, traffic_src = ncu_traffic(kern) if band == (0, hb) else (None, None)
    if rank == 0:
        ok = parity.get("decode") == "bit-exact"
        line = {
            "metric": METRIC, "value": value if ok else None, "unit": "Gpix/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_max, "higher_is_better": True,
            "scaling": scaling,
            "vs_baseline": None, "dtype": "int32", "data": "synthetic",
            "config": dict(workload_config(), bpp=round(st["bpp"], 4),
                           present_frac=round(st["present_frac"], 5),
                           kernel=kern, bands=[list(b) for b in bands] if world > 1 else [[0, hb]],
                           **({"test_hook": "BENCH_TEST_ONE_DEVICE: all ranks on cuda:0 over gloo, "
                                            "not a scaling measurement"} if one_dev else {})),
            "parity": parity,
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1),
                         "peak": peak, "unit": "GB/s",
                         "frac": round(achieved / peak, 4),
                         "traffic": traffic,
                         "traffic_source": traffic_src and (
                             traffic_src + " (ncu, DRAM bytes summed over "
                             "the step's kernels)"),
                         "peak_source": peak_kind,
                         "kernels": KERNELS[kern],
                         "alg_bytes_per_launch": int(alg),
                         "alg_bytes_note": "SURVEY 8d: offsets+SRV + int16 roots + RGB8 out, "
                                           "plus the prepared index read per step "
                                           "(entries, record flags, bitmap words and ranks)"},
            "index_build_ms": round(index_ms, 2),
            "per_rank_ms": per_rank,
            "e2e": e2e, "gpu_launches": args.steps * len(KERNELS[kern]),
            "clocks": clk.summary(),
            "cpu_baseline": cpu,
            "render": render,
            "random_access": random_access,
        }
        if not ok:
            line["error"] = "decoded field differs from the reference: value withheld"
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def parity_check(state, out, bands, scaling, world, rank, parallel):
    """sha256 of the decoded (S, T, H, W, 3) field vs the live reference's."""
    try:
        with open(REF_DECODE) as f:
            ref = json.load(f)
    except OSError:
        return {"decode": "unchecked", "why": "no reference golden"}
    import hashlib
    if hashlib.sha256(state.data).hexdigest() != ref["stream_sha256"]:
        return {"decode": "unchecked", "why": "stream differs from the golden's"}
    want = ref["k0"]["decode_all_sha256"]
    if world == 1:
        got = sha_host(out)
    elif scaling == "strong":
        full = parallel.gather_field(state, out, bands)     # band-major, all_gather_into_tensor
        got = sha_host(parallel.band_major_to_grid(full, state, bands)) if rank == 0 else None
    else:
        got = sha_host(out)
    res = {"decode": "bit-exact" if got == want or rank != 0 else "MISMATCH",
           "sha256": got, "reference_sha256": want,
           "reference": "tests/golden/cfg2_r4_decode_reference.json: live reference rlfc 0.1.0 "
                        "decode_image over all 289 views (tools/make_cfg2_decode_reference.py)"}
    return res


def render_measure(state, args, rl, world, rank):
    """cfg4: batches of 512x512 SlabPoses (s, t ~ U[0, S-1] x U[0, T-1]) x
    focal {image plane, 0.9, 1.12} x k {0, h}; poses sharded round-robin
    over the ranks (replicated stream).  Per cell: wall clock per batch
    (host pose prep + launches + sync, median of 7) and device time (CUDA
    events).  Parity: 6 views against the oracle's render of the oracle's
    decode (bit-exact)."""
    import torch
    import torch.distributed as dist
    hdr = state.header
    S, T, h = hdr.s_count, hdr.t_count, hdr.tree_height
    cells = []
    out = torch.empty((256, 512, 512, 3), dtype=torch.uint8, device="cuda")
    for batch in (1, 64, 256):
        for focal in (None, 0.9, 1.12):
            for k in (0, h):
                rng = np.random.default_rng(1000 * batch + 10 * k + (0 if focal is None else int(focal * 100)))
                allp = [rl.SlabPose(float(rng.uniform(0, S - 1)), float(rng.uniform(0, T - 1)), 512, 512, focal)
                        for _ in range(batch)]
                mine = allp[rank::world]
                o = out[:len(mine)]
                for _ in range(2):
                    if mine:
                        rl.render_views(state, mine, stop_level=k, out=o)
                torch.cuda.synchronize()
                wall = []
                for _ in range(7):
                    if world > 1:
                        dist.barrier()
                    t0 = time.perf_counter()
                    if mine:
                        rl.render_views(state, mine, stop_level=k, out=o)
                    torch.cuda.synchronize()
                    wall.append(time.perf_counter() - t0)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(5):
                    if mine:
                        rl.render_views(state, mine, stop_level=k, out=o)
                e1.record()
                torch.cuda.synchronize()
                dev_ms = e0.elapsed_time(e1) / 5
                w = statistics.median(wall)
                if world > 1:
                    t = torch.tensor([w, dev_ms], device="cuda")
                    dist.all_reduce(t, op=dist.ReduceOp.MAX)
                    w, dev_ms = float(t[0]), float(t[1])
                cells.append({"batch": batch, "focal_z": focal, "k": k,
                              "views_per_s": batch / w, "ms_per_batch": w * 1e3,
                              "device_ms_per_batch": dev_ms,
                              "device_views_per_s": batch / (dev_ms * 1e-3)})
    res = {"cells": cells, "view": "512x512 SlabPose, default geometry",
           "timing": "wall clock incl. host pose prep, sync per batch (median of 7); device = CUDA events",
           "sharding": f"poses round-robin over {world} rank(s), replicated stream"}
    head = next(c for c in cells if c["batch"] == 256 and c["focal_z"] is None and c["k"] == 0)
    res["views_per_s"] = head["views_per_s"]
    if rank == 0 and not args.no_cpu_baseline:
        res.update(render_parity_and_cpu(state, rl))
    return res


def render_parity_and_cpu(state, rl):
    from oracle import oracle
    hdr = state.header
    orc = oracle.OracleState(state.data)
    nth = oracle.lib().orc_nproc()
    field0, st0 = orc.decode_all(0, nthreads=nth)
    fieldh, sth = orc.decode_all(hdr.tree_height, nthreads=nth)
    assert st0 == 0 and sth == 0
    rng = np.random.default_rng(77)
    exact = 0
    cases = []
    for i, (focal, k) in enumerate([(None, 0), (0.9, 0), (1.12, 0), (None, 3), (0.9, 3), (1.12, 3),
                                   (None, 0), (1.12, 0)]):
        s, t = float(rng.uniform(0, hdr.s_count - 1)), float(rng.uniform(0, hdr.t_count - 1))
        k = min(k, hdr.tree_height)
        gpu = rl.render_view(state, rl.SlabPose(s, t, 512, 512, focal), stop_level=k)
        ref = orc.render_slab(s, t, 512, 512, focal_z=focal, stop_level=k,
                              field=field0 if k == 0 else fieldh)
        exact += int(np.array_equal(gpu, ref))
        cases.append([round(s, 4), round(t, 4), focal, k])
    # CPU baseline: the reference's per-view cost (decode the tap cameras,
    # then blend; renderer.py:212-276) in the C port, one view per thread
    import concurrent.futures as cf
    nv = 2 * nth
    poses = [(float(rng.uniform(0, hdr.s_count - 1)), float(rng.uniform(0, hdr.t_count - 1))) for _ in range(nv)]
    scratch = [np.zeros((hdr.s_count, hdr.t_count, hdr.height, hdr.width, 3), np.uint8) for _ in range(nth)]
    t0 = time.perf_counter()
    with cf.ThreadPoolExecutor(nth) as ex:
        list(ex.map(lambda ip: orc.render_slab_decoding(ip[1][0], ip[1][1], 512, 512,
                                                        scratch=scratch[ip[0] % nth]), enumerate(poses)))
    dt = time.perf_counter() - t0
    return {"parity": {"views_bit_exact": exact, "views_checked": len(cases), "poses": cases,
                       "against": "oracle render_slab of the oracle decode (renderer.py:233-276 order)"},
            "cpu_baseline": {"value": nv / dt, "unit": "views/s", "cores": nth, "kind": "port",
                             "sample": f"{nv} 512x512 slab views, tap cameras decoded per view then blended "
                                       "(reference per-view cost), one view per thread"}}


def e2e_measure(state, band, args, rl):
    import torch
    from paper_1805_06019_b200 import decoder
    res = decoder.HostPipeline(state, band)
    for _ in range(max(1, min(args.warmup, 2))):
        res.run()
    torch.cuda.synchronize()
    steps = max(1, min(args.steps, 5))
    t0 = time.perf_counter()
    for _ in range(steps):
        res.run()
    dt = (time.perf_counter() - t0) / steps
    hdr = state.header
    px = hdr.s_count * hdr.t_count * hdr.width * res.rows_px
    # this box's pinned-copy bandwidth: the PCIe floor of the step (the
    # D2H of the RGB field dominates; the bands overlap H2D, decode and D2H)
    bw = pcie_bandwidth()
    floor_ms = max(res.d2h_bytes / bw["d2h_gbs"], res.h2d_bytes / bw["h2d_gbs"]) / 1e6
    return {"value": px / dt / 1e9, "unit": "Gpix/s",
            "h2d_bytes_per_step": res.h2d_bytes,
            "d2h_bytes_per_step": res.d2h_bytes,
            "ms_per_step": dt * 1e3,
            "pcie": dict(bw, floor_ms=floor_ms, frac_of_floor=floor_ms / (dt * 1e3)),
            "path": "decoder.HostPipeline: pinned H2D of SRV+offsets+roots, "
                    "staged decode, pinned D2H of RGB; 8 block-row bands "
                    "pipelined over three CUDA streams (PCIe D2H-bound)"}


def pcie_bandwidth(nbytes=256 << 20, reps=8):
    """Pinned host <-> device copy bandwidth (GB/s) of one 256 MB buffer."""
    import torch
    h = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    out = {}
    for name, fn in (("h2d_gbs", lambda: d.copy_(h, non_blocking=True)),
                     ("d2h_gbs", lambda: h.copy_(d, non_blocking=True))):
        fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(reps):
            fn()
        torch.cuda.synchronize()
        out[name] = reps * nbytes / (time.perf_counter() - t0) / 1e9
    del h, d
    return out


def random_access_measure(state, rl):
    """Random-access block decode (decoder.decode_block path): 10^6-pick
    device-resident batches (throughput, CUDA events) and single-block calls
    through the public API (latency), picks from default_rng(7) as in the
    reference acceptance test."""
    import torch
    from paper_1805_06019_b200 import decoder
    hdr = state.header
    wb, hb = hdr.block_grid
    rng = np.random.default_rng(7)
    n = 1_000_000
    req = np.stack([rng.integers(0, hdr.s_count, n), rng.integers(0, hdr.t_count, n),
                    rng.integers(0, wb, n), rng.integers(0, hb, n),
                    rng.integers(0, 3, n), np.zeros(n, np.int64)], 1).astype(np.int32)
    dreq = torch.from_numpy(req).cuda()
    for _ in range(2):
        decoder.decode_blocks(state, dreq, raise_errors=False)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    reps = 5
    for _ in range(reps):
        decoder.decode_blocks(state, dreq, raise_errors=False)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    # Python ints, as a caller holds them (no numpy scalar conversions in
    # the timed loop)
    picks = [((s, t), (bx, by), c) for s, t, bx, by, c, _ in req[:2000].tolist()]
    for a in picks[:10]:
        rl.decode_block(state, *a)
    t0 = time.perf_counter()
    for a in picks:
        rl.decode_block(state, *a)
    lat = (time.perf_counter() - t0) / len(picks)
    return {"blocks_per_s": n / (ms * 1e-3), "batch": n, "ms_per_batch": ms,
            "decode_block_latency_us": lat * 1e6,
            "note": "cfg2 R4 stream, k=0, one CUDA thread per block request"}


CFG5 = dict(S=32, T=32, W=2048, H=2048, seed=7, h=3, B=4, shift=4, tp=16,
            tb=1000, codec="raw")


def make_stream_cfg5(cache_dir="/tmp/rlfc_cache"):
    """cfg5 (BASELINE configs[4]): 32x32x2048^2, 3-level tree, R4 params,
    produced band by band (producer.encode_synthetic_striped)."""
    from paper_1805_06019_b200 import encoder, lightfield, producer
    path = os.path.join(cache_dir, "cfg5_r4.rlfc")
    if os.path.exists(path):
        with open(path, "rb") as f:
            return f.read()
    t0 = time.time()
    params = encoder.EncodingParams(
        tree_height=CFG5["h"], block_size=CFG5["B"], quant_shift=CFG5["shift"],
        pixel_threshold=CFG5["tp"], block_threshold=CFG5["tb"],
        root_codec=CFG5["codec"])
    data, present = producer.encode_synthetic_striped(
        lightfield.SyntheticSpec(CFG5["S"], CFG5["T"], CFG5["W"], CFG5["H"],
                                 CFG5["seed"]), params, strip_rows=32)
    log(f"cfg5 stream {len(data)} B in {time.time() - t0:.0f}s, present {present}")
    os.makedirs(cache_dir, exist_ok=True)
    with open(path + ".tmp", "wb") as f:
        f.write(data)
    os.replace(path + ".tmp", path)
    return data


def run_cfg5(args):
    """Random-access block decode on the 32x32x2048^2 field: latency of
    single decode_block calls (10,000 picks, default_rng(7), as
    test_acceptance.py:165-177) and throughput of 10^6-pick device batches;
    plus one full-field decode (4.29 Gpix) for scale."""
    import torch
    import paper_1805_06019_b200 as rl
    from paper_1805_06019_b200 import decoder
    data = make_stream_cfg5()
    torch.zeros(1, device="cuda")                   # CUDA context outside the init timing
    torch.cuda.synchronize()
    t0 = time.time()
    state = rl.init(data)
    init_s = time.time() - t0
    hdr = state.header
    wb, hb = hdr.block_grid
    rng = np.random.default_rng(7)
    picks = np.stack([rng.integers(0, hdr.s_count, 10000), rng.integers(0, hdr.t_count, 10000),
                      rng.integers(0, wb, 10000), rng.integers(0, hb, 10000),
                      rng.integers(0, 3, 10000)], 1)
    calls = [((s, t), (bx, by), c) for s, t, bx, by, c in picks.tolist()]
    for a in calls[:50]:
        rl.decode_block(state, *a)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for a in calls:
        rl.decode_block(state, *a)
    lat_us = (time.perf_counter() - t0) / len(calls) * 1e6
    n = 1_000_000
    req = np.stack([rng.integers(0, hdr.s_count, n), rng.integers(0, hdr.t_count, n),
                    rng.integers(0, wb, n), rng.integers(0, hb, n),
                    rng.integers(0, 3, n), np.zeros(n, np.int64)], 1).astype(np.int32)
    dreq = torch.from_numpy(req).cuda()
    for _ in range(args.warmup):
        decoder.decode_blocks(state, dreq, raise_errors=False)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        decoder.decode_blocks(state, dreq, raise_errors=False)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    out = torch.empty((hdr.s_count, hdr.t_count, hdr.height, hdr.width, 3),
                      dtype=torch.uint8, device="cuda")
    decoder.decode_field(state, 0, out=out)
    torch.cuda.synchronize()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record()
    for _ in range(3):
        decoder.decode_field(state, 0, out=out, check=False)
    f1.record()
    torch.cuda.synchronize()
    field_ms = f0.elapsed_time(f1) / 3
    # CPU port: single-thread decode_block latency on 2,000 of the picks
    from oracle import oracle
    orc = oracle.OracleState(data)
    t0 = time.perf_counter()
    for p in picks[:2000]:
        orc.decode_block(int(p[0]), int(p[1]), int(p[2]), int(p[3]), int(p[4]), 0)
    cpu_us = (time.perf_counter() - t0) / 2000 * 1e6
    px = hdr.s_count * hdr.t_count * hdr.width * hdr.height
    line = {
        "metric": "random-access blocks/s (cfg5 32x32x2048^2, 10^6-pick batches)",
        "value": n / (ms * 1e-3), "unit": "blocks/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "int32", "data": "synthetic",
        "config": {"workload": "cfg5 random-access block decode, 32x32 views x 2048^2, h=3 B=4 R4 params, RAW roots",
                   "stream_bytes": len(data), "m_nodes": state.m_nodes,
                   "bpp": 8.0 * len(data) / px, "init_s": init_s},
        "decode_block_latency_us": lat_us,
        "full_field": {"gpix_per_s": px / (field_ms * 1e-3) / 1e9, "ms": field_ms},
        "cpu_baseline": {"value": 1e6 / cpu_us, "unit": "blocks/s", "cores": 1,
                         "kind": "port", "sample": "2,000 single decode_block picks, oracle C port",
                         "latency_us": cpu_us},
    }
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
