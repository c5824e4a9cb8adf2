"""Per-source-line instruction and stall shares from an ncu report (developer tool).

    ncu -i X.ncu-rep --page source --csv --print-source=cuda,sass > X.csv
    python profiles/source_hotspots.py X.csv [top]
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
cur, hdr, out = None, None, []
for r in rows:
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and r and r[0] and len(r) > 5 and r[2] == "-":
        ie = int(r[hdr.index("Instructions Executed")] or 0)
        st = int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
        out.append((ie, st, cur, r[0], r[1][:90]))
tot = sum(o[0] for o in out) or 1
tst = sum(o[1] for o in out) or 1
print(f"warp instructions {tot:.4g}, stall samples {tst}")
for ie, st, f, ln, src in sorted(out, reverse=True)[:top]:
    print(f"{ie / tot * 100:5.1f}% instr {st / tst * 100:5.1f}% samples  {f}:{ln}  {src.strip()}")
