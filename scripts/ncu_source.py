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
ap.add_argument("--wavefronts", action="store_true",
                help="instead: the instructions with most shared-memory wavefronts per unit")
args = ap.parse_args()
rows = list(csv.reader(open(args.csv)))
hdr = rows[1]
if args.wavefronts:
    iw, ii, ie, isr = (hdr.index("L1 Wavefronts Shared"), hdr.index("L1 Wavefronts Shared Ideal"),
                       hdr.index("Instructions Executed"), hdr.index("Source"))
    out = [(n, r[isr].strip(), int(r[ie] or 0), int(r[iw] or 0), int(r[ii] or 0))
           for n, r in enumerate(rows[2:]) if len(r) > iw and int(r[iw] or 0)]
    tot, ideal = sum(o[3] for o in out), sum(o[4] for o in out)
    print(f"shared-memory wavefronts {tot} = {tot / args.units:.1f} per unit "
          f"(ideal {ideal / args.units:.1f}: the rest are bank conflicts / same-address atomics)")
    for n, src, ex, w, idl in sorted(out, key=lambda o: -o[3])[:args.top]:
        print(f"sass {n:5d} {src[:52]:52s} exec/unit {ex / args.units:6.2f}  wavefronts/unit "
              f"{w / args.units:6.2f}  per instruction {w / max(ex, 1):5.2f}")
    raise SystemExit(0)
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
