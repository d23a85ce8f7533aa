"""Hand-run (GPU box): fixed cost of a search launch per config -- the kernel
on a one-block range [0, 4^S) -- against the full search."""
import sys; sys.path.insert(0, '.')
import numpy as np, torch, fmgen
import paper_1403_1313_b200 as pms
pms.build(); pms.load()
dev = torch.device("cuda", 0)
out = torch.zeros(1 << 20, dtype=torch.int32, device=dev)
cnt = torch.zeros(1, dtype=torch.int64, device=dev)
for ci in range(5):
    c = fmgen.BASELINE_CONFIGS[ci]
    s = torch.from_numpy(fmgen.generate_fm(c["n"], c["t"], c["l"], c["d"], 1)[0]).to(dev)
    with pms.Plan(c["n"], c["t"], c["l"], c["d"]) as plan:
        res = {}
        for name, hi in (("full", 4 ** c["l"]), ("one block", None), ("empty", 0)):
            ms = []
            for r in range(12):
                if name == "one block":
                    plan.execute_tensors(s, out, cnt, 0, 4 ** st.block_digits if r else 4 ** 5)
                else:
                    plan.execute_tensors(s, out, cnt, 0, hi)
                status, st = plan.wait()
                if r >= 2:
                    ms.append(st.search_ms)
            res[name] = (np.median(ms) * 1e3, st.pack_ms * 1e3)
        print(f"{c['name']:20s} S={st.block_digits} " + "  ".join(f"{k}: {v[0]:7.1f}us (pack {v[1]:.1f})" for k, v in res.items()), flush=True)
