"""Mean shrink of one fp16-split tcgen05 GEMM step vs the exact product, as a
function of K (the tensor core adds every MMA's dot product to the fp32
accumulator with truncation, so long K chains lose magnitude):
prints Re<got, ref> / <ref, ref> - 1 and the relative L2 error.

    python tools/rz_bias_probe.py
"""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2011_02621_b200 import _native as NV  # noqa: E402
from paper_2011_02621_b200.engine import ContractionPlan, NetworkSpec, PathExecutor  # noqa: E402


def probe(M, K, N, Z=2, kernel=NV.K_AUTO, tf32=False):
    edges = {(0, 1): K, (0, 2): M, (1, 2): N}
    legs = {0: [(0, 2), (0, 1)], 1: [(0, 1), (1, 2)], 2: [(0, 2), (1, 2)]}
    spec = NetworkSpec([0, 1, 2], edges, legs)
    g = torch.Generator(device="cuda")
    g.manual_seed(M + K + N)
    sites = {q: torch.randn((1,) + spec.site_dims(q), dtype=torch.complex64, device="cuda", generator=g) for q in range(3)}
    plan = ContractionPlan(spec, [0, 1, 2])
    ex = PathExecutor(plan, sites, dtype="complex64")
    d = ex._steps[0]
    acc = torch.randn(Z * M * K, dtype=torch.complex64, device="cuda", generator=g)
    out = torch.zeros(Z * M * N, dtype=torch.complex64, device="cuda")
    amax_in = torch.view_as_real(acc.reshape(Z, -1)).abs().reshape(Z, -1).amax(dim=1).contiguous()
    amax_out = torch.zeros(Z, dtype=torch.float32, device="cuda")
    d.Z, d.slices_per_b, d.s0 = Z, 1, 0
    d.acc, d.acc_zstride = acc.data_ptr(), M * K
    d.out, d.out_zstride = out.data_ptr(), M * N
    d.site.sel = None
    d.kernel = kernel
    d.amax_in, d.amax_out = (None if tf32 else amax_in.data_ptr()), amax_out.data_ptr()
    NV.check(NV.lib().tnc_step(C.byref(d), C.c_void_p(torch.cuda.current_stream().cuda_stream)), "tnc_step")
    torch.cuda.synchronize()
    site = ex.step_sites[0][0][0].reshape(K, N).to(torch.complex128)
    ref = acc.reshape(Z, M, K).to(torch.complex128) @ site
    got = out.reshape(Z, M, N).to(torch.complex128)
    shrink = (torch.sum(got * ref.conj()).real / torch.sum(ref * ref.conj()).real).item() - 1.0
    err = ((got - ref).norm() / ref.norm()).item()
    return shrink, err


if __name__ == "__main__":
    for K in (64, 256, 1024, 2048, 4096, 16384):
        M = 4096 if K <= 4096 else 2048
        s, e = probe(M, K, 128)
        print(f"K {K:6d}  N 128  shrink {s:+.3e}  rel L2 {e:.3e}  shrink/K {s / K:+.3e}")
    for K in (1024, 4096):
        s, e = probe(4096, K, 128, kernel=NV.K_GENERIC)
        print(f"K {K:6d}  SIMT    shrink {s:+.3e}  rel L2 {e:.3e}")
    # other tile shapes of the GEMM path: narrow (N <= 32), 4M N = 64, A-resident 4M (K <= 128, N >= 256),
    # single-CTA 3M (K < 512), 3xTF32 (no input bound)
    for (M, K, N, tf) in ((8192, 1024, 16, False), (8192, 1024, 64, False), (8192, 128, 256, False),
                          (8192, 256, 256, False), (8192, 1024, 16, True), (8192, 1024, 64, True),
                          (8192, 1024, 128, True), (8192, 8, 64, True)):
        s, e = probe(M, K, N, tf32=tf)
        print(f"M {M} K {K:6d} N {N:4d} {'tf32' if tf else 'f16 '} shrink {s:+.3e}  rel L2 {e:.3e}  shrink/K {s / K:+.3e}")
