"""Per-step summary of an ncu launch list of the decode path.

    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,\\
        dram__bytes_write.sum,sm__inst_executed.sum --clock-control none \\
        --csv --log-file launches.csv python tools/profile_decode.py
    python tools/ncu_summary.py launches.csv staged out.json

Takes the LAST complete decode step (one launch of each of the path's
kernels) and writes per-kernel time / DRAM bytes / instructions plus their
sums.  ncu serialises launches and flushes caches between them, so the
absolute times are cold-cache; the shares are what bench.py's live CUDA-event
numbers are compared against.
"""
import csv
import json
import sys

KERNELS = {"staged": ["k_payloads", "k_blend"],
           "fused": ["k_decode_field_tiled"]}


def main(path, kind, out):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, mi, vi, ii = (hdr.index(x) for x in
                      ("Kernel Name", "Metric Name", "Metric Value", "ID"))
    launches = {}
    for r in rows[1:]:
        d = launches.setdefault(int(r[ii]), {"name": r[ki]})
        d[r[mi]] = float(r[vi].replace(",", ""))
    names = KERNELS[kind]
    order = sorted(launches)
    step = {}
    for i in reversed(order):                       # last occurrence of each
        nm = next((n for n in names if n in launches[i]["name"]), None)
        if nm and nm not in step:
            step[nm] = launches[i]
        if len(step) == len(names):
            break
    per = {}
    for nm in names:
        d = step[nm]
        per[nm] = {"kernel": d["name"][:120],
                   "gpu_time_us": d["gpu__time_duration.sum"] / 1e3,
                   "dram_bytes_read": d["dram__bytes_read.sum"],
                   "dram_bytes_write": d["dram__bytes_write.sum"],
                   "inst_executed": d["sm__inst_executed.sum"]}
    tot_t = sum(p["gpu_time_us"] for p in per.values())
    for p in per.values():
        p["time_share"] = round(p["gpu_time_us"] / tot_t, 4)
    summary = {
        "path": kind,
        "capture": "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,"
                   "dram__bytes_write.sum,sm__inst_executed.sum "
                   "--clock-control none, tools/profile_decode.py (cfg2 R4), "
                   "last decode step",
        "source_file": path,
        "gpu_time_ms": tot_t / 1e3,
        "dram_bytes_read": sum(p["dram_bytes_read"] for p in per.values()),
        "dram_bytes_write": sum(p["dram_bytes_write"] for p in per.values()),
        "inst_executed": sum(p["inst_executed"] for p in per.values()),
        "alg_bytes": 1022727289,
        "kernels": per,
    }
    summary["dram_bytes_total"] = summary["dram_bytes_read"] + summary["dram_bytes_write"]
    with open(out, "w") as f:
        json.dump(summary, f, indent=1)
    print(json.dumps({k: v for k, v in summary.items() if k != "kernels"}))
    for nm, p in per.items():
        print(f"  {nm:12s} {p['gpu_time_us']:8.1f} us  share {p['time_share']:.3f}  "
              f"dram {(p['dram_bytes_read'] + p['dram_bytes_write']) / 1e6:8.1f} MB  "
              f"inst {p['inst_executed'] / 1e6:7.1f} M")


if __name__ == "__main__":
    main(*sys.argv[1:4])
