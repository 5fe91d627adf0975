"""Run one configs[1] sweep case (for ncu / quick timing):
    python tools/pair_case.py R K_LEGS N_LEGS B [iters] [seed|bench]"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2011_02621_b200.engine import PairPlan  # noqa: E402

r, k, n, B = (int(x) for x in sys.argv[1:5])
iters = int(sys.argv[5]) if len(sys.argv) > 5 else 5
# layout seed: 0, or "bench" for the sweep's own seed (the case index)
seed = 0
if len(sys.argv) > 6:
    seed = bench.sweep_cases().index((r, k, n, B)) if sys.argv[6] == "bench" else int(sys.argv[6])
perm, dims, pairs = bench.case_layout(r, k, n, seed=seed)
K, N = 4 ** k, 4 ** n
plan = PairPlan(dims, [4] * (k + n), pairs, dtype="complex64")
acc = torch.randn(B * 2 ** r * K, dtype=torch.complex64, device="cuda")
site = torch.randn(B * K * N, dtype=torch.complex64, device="cuda")
out = torch.empty(B * 2 ** r * N, dtype=torch.complex64, device="cuda")
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for i in range(iters):
    ev[0].record()
    plan(acc, site, out, B, 2 ** r * K, K * N, 2 ** r * N)
    ev[1].record()
    torch.cuda.synchronize()
by, fl = bench.case_traffic(r, k, n, B)
t = ev[0].elapsed_time(ev[1]) * 1e-3
print(f"case r={r} k={k} n={n} B={B} kernel={plan.kernel} {t*1e6:.1f} us {by/t/1e9:.0f} GB/s {fl/t/1e12:.1f} TF/s")
