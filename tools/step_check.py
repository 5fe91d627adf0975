"""Compare every step of a projected Sycamore plan between the default kernel
choice and the generic SIMT kernel on random accumulators (complex64).

Usage: python tools/step_check.py DEPTH [max_rank]"""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2011_02621_b200 import AmplitudeEngine, _native as NV, pattern_rqc, sycamore53_graph  # noqa: E402


def main():
    depth = int(sys.argv[1])
    mr = int(sys.argv[2]) if len(sys.argv) > 2 else 10
    graph, pats, _ = sycamore53_graph()
    c = pattern_rqc(graph, [pats[ch] for ch in "ABCDCDAB"], depth, seed=12)
    eng = AmplitudeEngine(c, dtype="complex64", max_rank=mr)
    ex, plan = eng.executor, eng.plan
    L = NV.lib()
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    Z = 2
    sel = {q: torch.tensor([0, 1], dtype=torch.int32, device="cuda") for q in range(53)}
    bad = 0
    for i, sp in enumerate(plan.steps):
        if sp.K * sp.N < 256:
            continue
        d = ex._steps[i]
        acc = torch.randn(Z * sp.M * sp.K, dtype=torch.complex64, device="cuda")
        outs = []
        for kern in (NV.K_AUTO, NV.K_GENERIC):
            out = torch.zeros(Z * sp.M * sp.N, dtype=torch.complex64, device="cuda")
            d.Z, d.slices_per_b, d.s0 = Z, 1, 0
            d.acc, d.acc_zstride = acc.data_ptr(), sp.M * sp.K
            d.out, d.out_zstride = out.data_ptr(), sp.M * sp.N
            d.site.sel = sel[sp.node].data_ptr() if ex.nvar[sp.node] > 1 else None
            d.kernel = kern
            NV.check(L.tnc_step(C.byref(d), st), "tnc_step")
            torch.cuda.synchronize()
            outs.append(out.cpu().numpy())
        d.kernel = NV.K_AUTO
        # direct reference: out[z, map(row, n)] = acc[z] (M x K) @ site[sel[z]] (K x N)
        dst = ex.step_sites[i][0]
        fd = [int(d.f_dim[j]) for j in range(d.nf)]
        fc = [int(d.f_cstride[j]) for j in range(d.nf)]
        f = np.arange(sp.M)
        oc = np.zeros(sp.M, dtype=np.int64)
        for j in range(d.nf - 1, -1, -1):
            oc += (f % fd[j]) * fc[j]
            f //= fd[j]
        off = torch.from_numpy(oc[:, None] + np.asarray(sp.c_noff, dtype=np.int64)[None, :]).cuda().reshape(-1)
        errs = []
        for kk in range(2):
            e2 = 0.0
            for z in range(Z):
                v = sel[sp.node][z].item() if ex.nvar[sp.node] > 1 else 0
                ref = acc[z * sp.M * sp.K:(z + 1) * sp.M * sp.K].reshape(sp.M, sp.K).to(torch.complex128) @ \
                    dst[v].reshape(sp.K, sp.N).to(torch.complex128)
                got = torch.from_numpy(outs[kk][z * sp.M * sp.N:(z + 1) * sp.M * sp.N]).cuda()[off].reshape(sp.M, sp.N)
                e2 = max(e2, ((got.to(torch.complex128) - ref).norm() / ref.norm()).item())
            errs.append(e2)
        print(f"   vs matmul: auto {errs[0]:.2e} generic {errs[1]:.2e}")
        err = np.linalg.norm(outs[0] - outs[1]) / np.linalg.norm(outs[1])
        flag = "BAD" if err > 1e-5 else ""
        bad += bool(flag)
        if flag and "--detail" in sys.argv:
            fd = [int(d.f_dim[j]) for j in range(d.nf)]
            fc = [int(d.f_cstride[j]) for j in range(d.nf)]
            rows = np.arange(sp.M)
            oc = np.zeros(sp.M, dtype=np.int64)
            f = rows.copy()
            for j in range(d.nf - 1, -1, -1):
                oc += (f % fd[j]) * fc[j]
                f //= fd[j]
            off = oc[:, None] + np.asarray(sp.c_noff, dtype=np.int64)[None, :]
            for z in range(Z):
                a = outs[0][z * sp.M * sp.N:(z + 1) * sp.M * sp.N][off]
                b = outs[1][z * sp.M * sp.N:(z + 1) * sp.M * sp.N][off]
                bad_m = np.abs(a - b) > 1e-3 * np.abs(b).max()
                rr, nn = np.nonzero(bad_m)
                print(f"   z={z}: {bad_m.sum()} bad of {bad_m.size}; rows {np.unique(rr // 128)[:20]} (tiles) n {np.unique(nn)[:40]}")
                if len(rr):
                    print("   sample", rr[:8], nn[:8], a[rr[:3], nn[:3]], b[rr[:3], nn[:3]])
        print(f"step {i:2d} M={sp.M:9d} K={sp.K:5d} N={sp.N:4d} contig={int(sp.c_rows_contig)} "
              f"ncontig={int(d.c_n_contig)} nf={d.nf} err={err:.2e} {flag}", flush=True)
    print("bad steps:", bad)


if __name__ == "__main__":
    main()
