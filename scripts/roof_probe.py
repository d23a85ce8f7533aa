"""Hand-run (GPU box): slice-family roofline microbenchmarks for each config."""
import sys; sys.path.insert(0, '.')
import torch, fmgen
import paper_1403_1313_b200 as pms
pms.build(); pms.load()
dev = torch.device("cuda", 0)
out = torch.zeros(1 << 20, dtype=torch.int32, device=dev)
cnt = torch.zeros(1, dtype=torch.int64, device=dev)
for ci in range(5):
    c = fmgen.BASELINE_CONFIGS[ci]
    s_np, _ = fmgen.generate_fm(c["n"], c["t"], c["l"], c["d"], 1)
    s = torch.from_numpy(s_np).to(dev)
    with pms.Plan(c["n"], c["t"], c["l"], c["d"]) as plan:
        for _ in range(3):
            plan.execute_tensors(s, out, cnt)
            st_, st = plan.wait()
        live = st.block_scans * (c['t'] - c['l'] + 1) / (st.search_ms * 1e-3)
        try:
            r0 = plan.roofline(0, 256); r1 = plan.roofline(1, 64)
            print(f"{c['name']:20s} S={st.block_digits} live {live/1e9:9.1f} Gtests/s  R_pass1 {r0['tests_per_s']/1e9:9.1f}  "
                  f"R_scan {r1['tests_per_s']/1e9:9.1f}  frac_scan {live/r1['tests_per_s']:.3f} frac_pass1 {live/r0['tests_per_s']:.3f} "
                  f"search {st.search_ms*1e3:.1f}us scans {st.block_scans}", flush=True)
        except pms.PmsError as e:
            print(c["name"], "roofline n/a:", e)
