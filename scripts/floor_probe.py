"""Hand-run probe (GPU box): the fixed cost of a search launch -- event time
of the slice search over 1 block vs the whole range, tables staged in shared
memory or read through L1/L2, at (9,2) and (13,3).
    python scripts/floor_probe.py"""
import sys
sys.path.insert(0, '.')
import numpy as np
import torch
import fmgen
import paper_1403_1313_b200 as pms

pms.load()
dev = torch.device("cuda", 0)
out = torch.zeros(1 << 20, dtype=torch.int32, device=dev)
cnt = torch.zeros(1, dtype=torch.int64, device=dev)
stream = torch.cuda.Stream()
for ci in (0, 2):
    c = fmgen.BASELINE_CONFIGS[ci]
    s_np, _ = fmgen.generate_fm(c["n"], c["t"], c["l"], c["d"], 1)
    s = torch.from_numpy(s_np).to(dev)
    for kw in ({}, {"table_global": 1}, {"seq_parallel": -1}, {"grid_ctas": 74}):
        for span in (1024, 16384, 4 ** c["l"]):
            with pms.Plan(c["n"], c["t"], c["l"], c["d"], pms.Launch(**kw)) as plan:
                ms = []
                with torch.cuda.stream(stream):
                    for r in range(23):
                        plan.execute_tensors(s, out, cnt, lo=0, hi=span, stream=stream)
                        st_, st = plan.wait()
                        assert st_ == 0
                        if r >= 3:
                            ms.append(st.search_ms)
            print(f"{c['name']:18s} {str(kw):24s} span={span:9d} S={st.block_digits} smem={st.table_in_smem} "
                  f"flags={st.mode_flags} search={np.median(ms)*1e3:7.2f}us min={min(ms)*1e3:7.2f}", flush=True)
