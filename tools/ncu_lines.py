"""Summarise an ncu source export (--page source --csv --print-source=cuda,sass)
per source line: warp-level instructions executed and stall samples."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
fname = None
out = []
hdr = None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) > 3 and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8 or not r[0]:
        continue
    try:
        inst = int(r[hdr.index("Instructions Executed")])
        samp = int(r[hdr.index("Warp Stall Sampling (All Samples)")])
    except (ValueError, IndexError):
        continue
    out.append((inst, samp, fname, r[0], r[1][:90]))
tot_i = sum(o[0] for o in out) or 1
tot_s = sum(o[1] for o in out) or 1
print(f"total warp-instructions {tot_i:,}  samples {tot_s:,}")
for inst, samp, f, ln, src in sorted(out, key=lambda o: -o[1])[:top]:
    print(f"{100*samp/tot_s:5.1f}%smp {100*inst/tot_i:5.1f}%ins {f}:{ln:>4} {src}")
