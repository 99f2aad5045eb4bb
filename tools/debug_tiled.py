"""Bisect helper: run the fused decode on every golden stream / stop level,
one launch at a time, and report the first failure."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from conftest import golden_names, load_golden, load_stream, sha  # noqa: E402
import paper_1805_06019_b200 as rl  # noqa: E402

names = sys.argv[1:] or golden_names()
for name in names:
    st = rl.init(load_stream(name))
    g = load_golden(name)
    for k in range(st.header.tree_height + 1):
        try:
            out, _ = rl.decode_field(st, k)
            torch.cuda.synchronize()
            ok = sha(out.cpu().numpy()) == str(g[f"all_k{k}_sha"])
            print(name, k, "ok" if ok else "MISMATCH", flush=True)
        except Exception as exc:  # noqa: BLE001
            print(name, k, "FAIL", type(exc).__name__, str(exc)[:80], flush=True)
            sys.exit(1)
