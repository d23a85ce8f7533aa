"""Hand-run timing sweep (GPU box): search-kernel time of each BASELINE config
under launch variants, via the plan API (CUDA events around the kernel).
    python scripts/sweep.py [--configs 0,1,2,3,4] [--reps 20] [--variants ...]
Variants are pms_launch fields as k=v,k=v; ';' separates variants."""
import argparse, json, sys
sys.path.insert(0, '.')
import numpy as np
import torch
import fmgen
import paper_1403_1313_b200 as pms

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="0,1,2,3,4")
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--seed", type=int, default=1)
ap.add_argument("--variants", default="algo=3;algo=2")
args = ap.parse_args()
pms.build(); pms.load()
dev = torch.device("cuda", 0)
out = torch.zeros(1 << 20, dtype=torch.int32, device=dev)
cnt = torch.zeros(1, dtype=torch.int64, device=dev)
stream = torch.cuda.Stream()
for ci in [int(x) for x in args.configs.split(",")]:
    c = fmgen.BASELINE_CONFIGS[ci]
    s_np, _ = fmgen.generate_fm(c["n"], c["t"], c["l"], c["d"], args.seed)
    s = torch.from_numpy(s_np).to(dev)
    gold = json.load(open(f"tests/golden/bj{ci}_seed{args.seed}.json"))["codes"]
    for v in args.variants.split(";"):
        kw = {k: int(x) for k, x in (p.split("=") for p in v.split(",") if p)}
        with pms.Plan(c["n"], c["t"], c["l"], c["d"], pms.Launch(**kw)) as plan:
            ms, pk = [], []
            with torch.cuda.stream(stream):
                for r in range(args.reps + 2):
                    plan.execute_tensors(s, out, cnt, stream=stream)
                    st_, st = plan.wait()
                    assert st_ == 0
                    if r >= 2:
                        ms.append(st.search_ms); pk.append(st.pack_ms)
            codes = sorted(out[:int(cnt.item())].cpu().numpy().astype(np.uint32).tolist())
        print(f"{c['name']:20s} {v:28s} algo={st.algo} S={st.block_digits} grid={st.grid}x{st.block} "
              f"smem={st.table_in_smem} search={np.median(ms)*1e3:9.1f}us (min {min(ms)*1e3:8.1f}) "
              f"pack={np.median(pk)*1e3:6.1f}us scans={st.block_scans} parity={codes == gold}",
              flush=True)
