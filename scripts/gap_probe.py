"""Hand-run probe (GPU box): per BASELINE config, the pre-pass / search /
whole-step event times with the search timed alone (an event between the two
kernels) and with the two overlapped (pms_launch.overlap_prepass), so the
launch gap between the kernels is visible.
    python scripts/gap_probe.py [--configs 0,1,2,3] [--reps 30] [--tag NAME]"""
import argparse, json, sys
sys.path.insert(0, '.')
import numpy as np
import torch
import fmgen
import paper_1403_1313_b200 as pms

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="0,1,2,3")
ap.add_argument("--reps", type=int, default=30)
ap.add_argument("--tag", default="")
ap.add_argument("--variants", default="")
args = ap.parse_args()
pms.load()
dev = torch.device("cuda", 0)
out = torch.zeros(1 << 20, dtype=torch.int32, device=dev)
cnt = torch.zeros(1, dtype=torch.int64, device=dev)
stream = torch.cuda.Stream()
for ci in [int(x) for x in args.configs.split(",")]:
    c = fmgen.BASELINE_CONFIGS[ci]
    s_np, _ = fmgen.generate_fm(c["n"], c["t"], c["l"], c["d"], 1)
    s = torch.from_numpy(s_np).to(dev)
    gold = json.load(open(f"tests/golden/bj{ci}_seed1.json"))["codes"]
    for v in (args.variants.split(";") if args.variants else [""]):
        kw = {k: int(x) for k, x in (p.split("=") for p in v.split(",") if p)}
        row = {"tag": args.tag, "config": c["name"], "variant": v}
        for ov in (0, 1):
            with pms.Plan(c["n"], c["t"], c["l"], c["d"], pms.Launch(overlap_prepass=ov, **kw)) as plan:
                se, pk, tot = [], [], []
                with torch.cuda.stream(stream):
                    for r in range(args.reps + 3):
                        plan.execute_tensors(s, out, cnt, stream=stream)
                        st_, st = plan.wait()
                        assert st_ == 0
                        if r >= 3:
                            se.append(st.search_ms); pk.append(st.pack_ms); tot.append(st.total_ms)
                codes = sorted(out[:int(cnt.item())].cpu().numpy().astype(np.uint32).tolist())
            key = "ovl" if ov else "sep"
            row[key] = {"search_us": round(float(np.median(se)) * 1e3, 2),
                        "pack_us": round(float(np.median(pk)) * 1e3, 2),
                        "step_us": round(float(np.median(tot)) * 1e3, 2),
                        "step_min_us": round(float(np.min(tot)) * 1e3, 2),
                        "parity": codes == gold}
        print(json.dumps(row), flush=True)
