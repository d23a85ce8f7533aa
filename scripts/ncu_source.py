"""Per-segment instruction breakdown of a kernel from an ncu source page
(`ncu -i REP --page source --csv --print-source sass > F.csv`): consecutive
SASS instructions with the same execution count form a segment; prints each
segment's warp instructions per unit (e.g. per block scan) and stall samples.

    python scripts/ncu_source.py F.csv --units N [--top 25]
"""
import argparse
import csv

ap = argparse.ArgumentParser()
ap.add_argument("csv")
ap.add_argument("--units", type=float, required=True)
ap.add_argument("--top", type=int, default=25)
args = ap.parse_args()
rows = list(csv.reader(open(args.csv)))
hdr = rows[1]
ix, isrc, iex, ismp = (hdr.index("Address"), hdr.index("Source"), hdr.index("Instructions Executed"),
                      hdr.index("Warp Stall Sampling (All Samples)"))
ins = [(i, r[isrc].strip(), int(r[iex] or 0), int(r[ismp] or 0)) for i, r in enumerate(rows[2:]) if len(r) > iex]
segs, cur = [], None
for i, src, ex, smp in ins:
    if cur and cur["ex"] == ex and i == cur["end"] + 1:
        cur["end"] = i; cur["n"] += 1; cur["smp"] += smp; cur["ops"].append(src.split()[0] if src else "?")
    else:
        cur = {"start": i, "end": i, "ex": ex, "n": 1, "smp": smp, "ops": [src.split()[0] if src else "?"]}
        segs.append(cur)
tot = sum(s["ex"] * s["n"] for s in segs)
tsmp = sum(s["smp"] for s in segs) or 1
print(f"total warp instructions {tot} = {tot / args.units:.1f} per unit; stall samples {tsmp}")
for s in sorted(segs, key=lambda s: -s["ex"] * s["n"])[: args.top]:
    per = s["ex"] * s["n"] / args.units
    print(f"sass {s['start']:5d}-{s['end']:5d} x {s['ex']:9d} ({s['n']:3d} instr) = {per:6.1f}/unit "
          f"samples {100 * s['smp'] / tsmp:5.1f}%  {' '.join(s['ops'][:14])}")
