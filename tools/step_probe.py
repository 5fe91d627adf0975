"""Time one large engine step acc[M, K] x S[K, N] (complex64) in isolation.

Usage: python tools/step_probe.py M K N [reps]
Network 0-1-2 (edges K, M, N); step 1 is the probed step.  Prints the step
time from CUDA events around a bare tnc_step call."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2011_02621_b200 import _native as NV  # noqa: E402
from paper_2011_02621_b200.engine import ContractionPlan, NetworkSpec, PathExecutor  # noqa: E402


def main():
    M, K, N = (int(x) for x in sys.argv[1:4])
    reps = int(sys.argv[4]) if len(sys.argv) > 4 else 10
    edges = {(0, 1): K, (0, 2): M, (1, 2): N}
    legs = {0: [(0, 2), (0, 1)], 1: [(0, 1), (1, 2)], 2: [(0, 2), (1, 2)]}
    spec = NetworkSpec([0, 1, 2], edges, legs)
    g = torch.Generator(device="cuda")
    g.manual_seed(0)
    sites = {q: torch.randn((1,) + spec.site_dims(q), dtype=torch.complex64, device="cuda", generator=g) for q in range(3)}
    plan = ContractionPlan(spec, [0, 1, 2])
    ex = PathExecutor(plan, sites, dtype="complex64")
    amp = torch.zeros(1, dtype=torch.complex64, device="cuda")
    ex.run(None, 1, amp)
    sp = plan.steps[0]
    L = NV.lib()
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    d = ex._steps[0]
    for _ in range(2):
        NV.check(L.tnc_step(C.byref(d), st), "tnc_step")
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        NV.check(L.tnc_step(C.byref(d), st), "tnc_step")
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / reps * 1e-3
    by = (sp.M * sp.K + sp.M * sp.N) * 8
    fl = 8 * sp.M * sp.K * sp.N
    msg = ""
    if "--check" in sys.argv:
        acc = torch.randn(sp.M * sp.K, dtype=torch.complex64, device="cuda")
        out = torch.zeros(sp.M * sp.N, dtype=torch.complex64, device="cuda")
        d.acc, d.out = acc.data_ptr(), out.data_ptr()
        NV.check(L.tnc_step(C.byref(d), st), "tnc_step")
        torch.cuda.synchronize()
        site = ex.step_sites[0][0][0].reshape(sp.K, sp.N).to(torch.complex128)
        ref = acc.reshape(sp.M, sp.K).to(torch.complex128) @ site
        diff = (out.reshape(sp.M, sp.N).to(torch.complex128) - ref).abs()
        bad = diff > 1e-3 * ref.abs().max()
        msg = f" rel_err {(diff.norm() / ref.norm()).item():.2e} bad {int(bad.sum())}"
        if int(bad.sum()):
            rr = torch.nonzero(bad)
            msg += f" tiles {sorted(set((rr[:, 0] // 128).tolist()))[:10]} ntile {sorted(set((rr[:, 1] // 64).tolist()))}"
            msg += f" rows%128 {sorted(set((rr[:, 0] % 128).tolist()))[:40]} cols {sorted(set(rr[:, 1].tolist()))[:70]}"
    print(f"M={sp.M} K={sp.K} N={sp.N} contig={int(sp.c_rows_contig)}: {t * 1e6:.1f} us "
          f"{by / t / 1e9:.0f} GB/s {fl / t / 1e12:.1f} TF/s{msg}")


if __name__ == "__main__":
    main()
