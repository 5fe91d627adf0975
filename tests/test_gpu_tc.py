"""Tensor-core (tcgen05 3xTF32 / fp16-split) contraction paths and the SIMT
step kernels vs the CPU oracle and complex128 references."""

from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]

import tn_oracle as O

pytestmark = pytest.mark.gpu


def rel_l2(got, ref):
    return float(np.linalg.norm(np.asarray(got) - ref) / np.linalg.norm(ref))


@pytest.mark.parametrize("r,k,n,B,ascale,bscale", [
    (7, 1, 2, 2, 1.0, 1.0), (7, 2, 2, 3, 1.0, 1.0), (8, 3, 3, 2, 1.0, 1.0), (9, 1, 3, 2, 1.0, 1.0),
    (9, 3, 2, 3, 1.0, 1.0), (10, 2, 3, 1, 1.0, 1.0), (11, 3, 3, 1, 1.0, 1.0), (7, 3, 2, 1, 1.0, 1.0),
    (8, 3, 1, 3, 1.0, 1.0), (9, 3, 1, 1, 1.0, 1.0),
    # fp16-split path: arbitrary operand scales and a wide per-row dynamic range
    (9, 2, 2, 3, 1e-25, 1e20), (8, 3, 2, 2, 3e12, 1e-9), (10, 2, 3, 2, 1e-22, 1e-8), (8, 3, 3, 2, 7e-3, 5e4)])
@pytest.mark.parametrize("f16", ["0", "1"])
@pytest.mark.parametrize("bulk", ["1", "0"])
def test_tc_pair_matches_oracle(r, k, n, B, ascale, bscale, f16, bulk, monkeypatch):
    import torch

    monkeypatch.setenv("TNC_TC_F16", f16)          # opt-in fp16-split variant of k_tc_c64 (read per launch)
    monkeypatch.setenv("TNC_TC_BULKOUT", bulk)     # N = 16 cases: bulk-store epilogue, or the STG path

    from paper_2011_02621_b200.engine import PairPlan

    rng = np.random.default_rng(1000 + r * 100 + k * 10 + n)
    perm = list(rng.permutation(r + k))
    dims = [2 if x < r else 4 for x in perm]
    size = int(np.prod(dims))
    acc = ((rng.standard_normal((B, size)) + 1j * rng.standard_normal((B, size))) / np.sqrt(2))
    if ascale != 1.0:
        acc = acc * np.exp(rng.uniform(-6, 6, (B, size)))      # rows spanning ~5 decades
    acc = (acc * ascale).astype(np.complex64)
    site = ((rng.standard_normal((2,) + (4,) * (k + n)) + 1j * rng.standard_normal((2,) + (4,) * (k + n))) / 2
            * bscale).astype(np.complex64)
    bits = rng.integers(0, 2, B)
    shared_pos = sorted((i for i, x in enumerate(perm) if x >= r), key=lambda i: perm[i])
    pairs = [(p, j) for j, p in enumerate(shared_pos)]
    plan = PairPlan(dims, [4] * (k + n), pairs, dtype="complex64")
    K, N = 4 ** k, 4 ** n
    if K * N >= 256 and K >= 8:                  # K <= 4 stays on the SIMT column kernel
        assert plan.kernel.startswith("tcgen05-3x")
    ta = torch.from_numpy(acc).cuda()
    sb = torch.from_numpy(np.ascontiguousarray(site[bits].reshape(B, -1))).cuda()
    out = torch.empty((B, size // K * N), dtype=torch.complex64, device="cuda")
    plan(ta, sb, out, B, size, K * N, size // K * N)
    torch.cuda.synchronize()
    ref = O.sweep_step(acc.astype(np.complex128), perm, r, k, site.astype(np.complex128), bits)
    err = rel_l2(out.cpu().numpy(), ref)
    assert err <= 2e-6, err


@pytest.mark.parametrize("r,k,n,B,seed", [(12, 2, 2, 2, "bench:16,2,2,256"), (12, 2, 3, 2, "bench:16,2,3,16"),
                                         (12, 3, 3, 1, "bench:16,3,3,16"), (12, 3, 1, 2, "bench:16,3,1,1")])
@pytest.mark.parametrize("noxor", [False, True])
def test_tc_pair_sweep_layouts(r, k, n, B, seed, noxor, monkeypatch):
    """k_tc_c64 on the sweep's own leg permutations (bench.case_layout seeds), whose
    staged-tile reads use the per-row k-slot XOR (TcDesc::kx_row) -- and with it off"""
    import torch

    import bench
    from paper_2011_02621_b200.engine import PairPlan

    if noxor:
        monkeypatch.setenv("TNC_TC_NOXOR", "1")
    case = tuple(int(x) for x in seed.split(":")[1].split(","))
    perm, dims, pairs = bench.case_layout(case[0], case[1], case[2], bench.sweep_cases()[0].index(case))
    # keep the innermost legs (the tile's row/k bank pattern) and drop outer row legs
    drop = case[0] - r
    keep = [i for i, x in enumerate(perm) if not (x < case[0] and sum(1 for y in perm[:i] if y < case[0]) < drop)]
    perm = [perm[i] for i in keep]
    order = sorted(range(len(perm)), key=lambda i: perm[i])
    rank = {i: j for j, i in enumerate(order)}
    perm = [rank[i] for i in range(len(perm))]
    dims = [2 if x < r else 4 for x in perm]
    shared_pos = sorted((i for i, x in enumerate(perm) if x >= r), key=lambda i: perm[i])
    pairs = [(p, j) for j, p in enumerate(shared_pos)]
    rng = np.random.default_rng(7)
    size = int(np.prod(dims))
    acc = ((rng.standard_normal((B, size)) + 1j * rng.standard_normal((B, size))) / np.sqrt(2)).astype(np.complex64)
    site = ((rng.standard_normal((2,) + (4,) * (k + n)) + 1j * rng.standard_normal((2,) + (4,) * (k + n))) / 2
            ).astype(np.complex64)
    bits = rng.integers(0, 2, B)
    plan = PairPlan(dims, [4] * (k + n), pairs, dtype="complex64")
    K, N = 4 ** k, 4 ** n
    assert plan.kernel.startswith("tcgen05-3x")
    ta = torch.from_numpy(acc).cuda()
    sb = torch.from_numpy(np.ascontiguousarray(site[bits].reshape(B, -1))).cuda()
    out = torch.empty((B, size // K * N), dtype=torch.complex64, device="cuda")
    plan(ta, sb, out, B, size, K * N, size // K * N)
    torch.cuda.synchronize()
    ref = O.sweep_step(acc.astype(np.complex128), perm, r, k, site.astype(np.complex128), bits)
    assert rel_l2(out.cpu().numpy(), ref) <= 2e-6


def test_tc_engine_step_contiguous():
    """Engine-layout step (accumulator rows contiguous) through tnc_step."""
    import torch

    from paper_2011_02621_b200 import AmplitudeEngine, pattern_rqc, sycamore53_graph

    graph, pats, _ = sycamore53_graph()
    seq = [pats[ch] for ch in "ABCDCDAB"]
    c = pattern_rqc(graph, seq, 5, seed=4)
    rng = np.random.default_rng(2)
    outs = ["".join(rng.choice(["0", "1"], 53)) for _ in range(6)]
    e128 = AmplitudeEngine(c, dtype="complex128", max_rank=10)
    ref = e128.amplitudes(outs)
    e64 = AmplitudeEngine(c, dtype="complex64", max_rank=10)
    kn = [(sp.K, sp.N, sp.M, sp.c_rows_contig) for sp in e64.plan.steps]
    got = e64.amplitudes(outs)
    assert rel_l2(got, ref) <= 1e-4, (rel_l2(got, ref), kn)


@pytest.mark.parametrize("dtype,tol,scaled_tol", [("complex128", 1e-12, 1e-15), ("complex64", 1e-4, 2e-7)])
@pytest.mark.parametrize("V", [1, 3])
def test_engine_tensor_core_steps(dtype, tol, scaled_tol, V):
    """Engine steps with K*N >= 256 run on the tensor cores (DMMA for
    complex128, tcgen05 3xTF32 for complex64); chain 0-1-2 plus a closing
    edge, checked against the numpy oracle per variant.  The amplitudes of
    this random network cancel heavily (|amp| ~ 1e-3 of sum|terms|), so the
    complex64 check is the north-star relative bound plus an absolute error
    bound scaled by the contraction of |sites| (fp32 accumulation level)."""
    import torch

    from paper_2011_02621_b200.engine import ContractionPlan, NetworkSpec, PathExecutor

    rng = np.random.default_rng(7 + V)
    edges = {(0, 1): 64, (1, 2): 32, (0, 2): 128, (2, 3): 4, (0, 3): 2}
    legs = {0: [(0, 1), (0, 2), (0, 3)], 1: [(0, 1), (1, 2)], 2: [(0, 2), (1, 2), (2, 3)], 3: [(0, 3), (2, 3)]}
    spec = NetworkSpec([0, 1, 2, 3], edges, legs)
    sites = {}
    for q in range(4):
        dims = spec.site_dims(q)
        sites[q] = (rng.standard_normal((V,) + dims) + 1j * rng.standard_normal((V,) + dims)) / np.sqrt(np.prod(dims))
    plan = ContractionPlan(spec, [0, 1, 2, 3])
    assert any(sp.K * sp.N >= 256 and sp.M % 128 == 0 for sp in plan.steps)
    ex = PathExecutor(plan, {q: torch.from_numpy(sites[q]) for q in range(4)}, dtype=dtype)
    B = 4
    bits = rng.integers(0, V, (B, 4)).astype(np.int32)
    sel = {q: torch.from_numpy(np.ascontiguousarray(bits[:, q])).cuda() for q in range(4)}
    amp = torch.zeros(B, dtype=ex.tdtype, device="cuda")
    ex.run(sel, B, amp)
    got = amp.cpu().numpy().astype(np.complex128)
    ref = np.array([O.contract_along_path({q: (sites[q][bits[b, q]], legs[q]) for q in range(4)}, [0, 1, 2, 3])[0]
                    for b in range(B)])
    scale = np.array([O.contract_along_path({q: (np.abs(sites[q][bits[b, q]]), legs[q]) for q in range(4)},
                                            [0, 1, 2, 3])[0] for b in range(B)])
    assert rel_l2(got, ref) <= tol
    assert np.max(np.abs(got - ref) / np.abs(scale)) <= scaled_tol


@pytest.mark.parametrize("depth", [6, 7])
def test_tc_gemm_engine_sycamore(depth):
    """53-qubit Sycamore network (projected, cap 10): large due-ordered steps
    with interleaved result layouts go through the tcgen05 GEMM path; complex64
    amplitudes agree with the complex128 engine to the 1e-4 north-star bound."""
    from paper_2011_02621_b200 import AmplitudeEngine, pattern_rqc, sycamore53_graph

    graph, pats, _ = sycamore53_graph()
    c = pattern_rqc(graph, [pats[ch] for ch in "ABCDCDAB"], depth, seed=12)
    rng = np.random.default_rng(depth)
    outs = ["".join(rng.choice(["0", "1"], 53)) for _ in range(4)]
    e64 = AmplitudeEngine(c, dtype="complex64", max_rank=10)
    big = [sp for sp in e64.plan.steps if sp.K * sp.N >= 256 and not sp.c_rows_contig]
    assert big, "expected interleaved large steps"
    ref = AmplitudeEngine(c, dtype="complex128", max_rank=10).amplitudes(outs)
    got = e64.amplitudes(outs)
    assert rel_l2(got, ref) <= 1e-4, rel_l2(got, ref)


@pytest.mark.parametrize("M,K,N", [(128, 64, 4), (128, 1024, 4), (256, 4096, 64), (128, 4096, 128), (384, 256, 24)])
def test_tc_gemm_scaled_precision(M, K, N):
    """One large step acc[M, K] x S[K, N] (tcgen05 GEMM path), closed against
    S2[M, N]: error relative to the contraction of |sites| stays at the fp32
    accumulation level (3xTF32 products, fp32 tensor-core accumulation)."""
    import torch

    from paper_2011_02621_b200.engine import ContractionPlan, NetworkSpec, PathExecutor

    rng = np.random.default_rng(M + K + N)
    edges = {(0, 1): K, (0, 2): M, (1, 2): N}
    legs = {0: [(0, 1), (0, 2)], 1: [(0, 1), (1, 2)], 2: [(0, 2), (1, 2)]}
    spec = NetworkSpec([0, 1, 2], edges, legs)
    sites = {q: (rng.standard_normal((1,) + spec.site_dims(q)) + 1j * rng.standard_normal((1,) + spec.site_dims(q)))
             .astype(np.complex64).astype(np.complex128) for q in range(3)}
    plan = ContractionPlan(spec, [0, 1, 2])
    assert (plan.steps[0].M, plan.steps[0].K, plan.steps[0].N) == (M, K, N)
    ex = PathExecutor(plan, {q: torch.from_numpy(sites[q]) for q in range(3)}, dtype="complex64")
    amp = torch.zeros(1, dtype=ex.tdtype, device="cuda")
    ex.run(None, 1, amp)
    got = complex(amp.cpu().numpy()[0])
    ref = O.contract_along_path({q: (sites[q][0], legs[q]) for q in range(3)}, [0, 1, 2])[0]
    scale = O.contract_along_path({q: (np.abs(sites[q][0]), legs[q]) for q in range(3)}, [0, 1, 2])[0]
    assert abs(got - ref) / abs(scale) <= 2e-7


@pytest.mark.parametrize("M,K,N,scale,sscale", [(8192, 128, 256, 1.0, 1.0), (16384, 256, 128, 3e-21, 1.0),
                                                 (8192, 16, 128, 7e12, 1.0), (32768, 16, 16, 1.0, 1.0),
                                                 (8192, 64, 24, 1e-3, 1.0),
                                                 # both scales large: their product leaves the fp32 range
                                                 (8192, 128, 256, 1e-25, 1e-12), (16384, 16, 16, 1e-24, 1e-13),
                                                 # 128-wide 3M (Gauss) tiles, K > 128; round-robin item order
                                                 (8192, 256, 256, 1.0, 1.0), (4096, 512, 128, 3e-21, 1.0),
                                                 (2048, 1024, 384, 1e-25, 1e-12), (4096, 256, 200, 7e12, 1.0),
                                                 (1536, 2048, 1024, 1.0, 1e-3),
                                                 # CTA-pair kernel (K >= 512): odd row-tile count (last pair half
                                                 # empty), ragged N, rows past M
                                                 (3200, 512, 384, 1.0, 1.0), (3100, 1024, 200, 3e-21, 1e-3),
                                                 (8192, 512, 128, 7e12, 1.0)])
def test_tc_gemm_f16_split_step(M, K, N, scale, sscale):
    """fp16-split tcgen05 GEMM (a step given amax_in): one step acc[M, K] x
    S[K, N] on inputs spanning ~12 decades around an arbitrary overall scale
    matches the complex128 product to the 3xTF32 level (relative L2 <= 2e-6),
    and amax_out records max |re|, |im| of the result."""
    import ctypes as C

    import torch

    from paper_2011_02621_b200 import _native as NV
    from paper_2011_02621_b200.engine import ContractionPlan, NetworkSpec, PathExecutor

    edges = {(0, 1): K, (0, 2): M, (1, 2): N}
    legs = {0: [(0, 2), (0, 1)], 1: [(0, 1), (1, 2)], 2: [(0, 2), (1, 2)]}
    spec = NetworkSpec([0, 1, 2], edges, legs)
    g = torch.Generator(device="cuda")
    g.manual_seed(M + K + N)
    sites = {q: torch.randn((1,) + spec.site_dims(q), dtype=torch.complex64, device="cuda", generator=g) for q in range(3)}
    sites[1] = sites[1] * sscale
    plan = ContractionPlan(spec, [0, 1, 2])
    sp = plan.steps[0]
    assert (sp.M, sp.K, sp.N) == (M, K, N)
    ex = PathExecutor(plan, sites, dtype="complex64")
    d = ex._steps[0]
    Z = 2
    mag = torch.exp(torch.empty(Z * M * K, device="cuda").uniform_(-14, 14, generator=g))
    acc = (torch.randn(Z * M * K, dtype=torch.complex64, device="cuda", generator=g) * mag * scale).to(torch.complex64)
    out = torch.zeros(Z * M * N, dtype=torch.complex64, device="cuda")
    amax_in = torch.view_as_real(acc.reshape(Z, -1)).abs().reshape(Z, -1).amax(dim=1).contiguous()
    amax_out = torch.zeros(Z, dtype=torch.float32, device="cuda")
    d.Z, d.slices_per_b, d.s0 = Z, 1, 0
    d.acc, d.acc_zstride = acc.data_ptr(), M * K
    d.out, d.out_zstride = out.data_ptr(), M * N
    d.site.sel = None
    d.amax_in, d.amax_out = amax_in.data_ptr(), amax_out.data_ptr()
    L = NV.lib()
    NV.check(L.tnc_step(C.byref(d), C.c_void_p(torch.cuda.current_stream().cuda_stream)), "tnc_step")
    torch.cuda.synchronize()
    site = ex.step_sites[0][0][0].reshape(K, N).to(torch.complex128)
    ref = acc.reshape(Z, M, K).to(torch.complex128) @ site
    got = out.reshape(Z, M, N).to(torch.complex128)
    err = ((got - ref).norm() / ref.norm()).item()
    assert err <= 2e-6, err
    want = torch.view_as_real(out.reshape(Z, -1)).abs().reshape(Z, -1).amax(dim=1)
    assert torch.equal(amax_out, want), (amax_out, want)


@pytest.mark.parametrize("M,K,N", [(8192, 8192, 128), (4096, 5120, 256), (2048, 16384, 128)])
def test_tc_gemm_long_k_segments(M, K, N):
    """K > 2048 on the CTA-pair kernel: the K loop leaves the tensor core every
    2048 complex (fp32 round-to-nearest adds of the segment sums), so the
    round-toward-zero accumulation inside the tensor core does not grow with K
    (unsegmented: 1.5e-5 at K = 8192, 2.9e-5 at 16384); ragged last segment;
    amax_out tracks the final sums."""
    import ctypes as C

    import torch

    from paper_2011_02621_b200 import _native as NV
    from paper_2011_02621_b200.engine import ContractionPlan, NetworkSpec, PathExecutor

    edges = {(0, 1): K, (0, 2): M, (1, 2): N}
    legs = {0: [(0, 2), (0, 1)], 1: [(0, 1), (1, 2)], 2: [(0, 2), (1, 2)]}
    spec = NetworkSpec([0, 1, 2], edges, legs)
    g = torch.Generator(device="cuda")
    g.manual_seed(M + K + N)
    sites = {q: torch.randn((1,) + spec.site_dims(q), dtype=torch.complex64, device="cuda", generator=g) for q in range(3)}
    plan = ContractionPlan(spec, [0, 1, 2])
    ex = PathExecutor(plan, sites, dtype="complex64")
    d = ex._steps[0]
    Z = 2
    acc = torch.randn(Z * M * K, dtype=torch.complex64, device="cuda", generator=g)
    out = torch.zeros(Z * M * N, dtype=torch.complex64, device="cuda")
    amax_in = torch.view_as_real(acc.reshape(Z, -1)).abs().reshape(Z, -1).amax(dim=1).contiguous()
    amax_out = torch.zeros(Z, dtype=torch.float32, device="cuda")
    d.Z, d.slices_per_b, d.s0 = Z, 1, 0
    d.acc, d.acc_zstride = acc.data_ptr(), M * K
    d.out, d.out_zstride = out.data_ptr(), M * N
    d.site.sel = None
    d.amax_in, d.amax_out = amax_in.data_ptr(), amax_out.data_ptr()
    NV.check(NV.lib().tnc_step(C.byref(d), C.c_void_p(torch.cuda.current_stream().cuda_stream)), "tnc_step")
    torch.cuda.synchronize()
    site = ex.step_sites[0][0][0].reshape(K, N).to(torch.complex128)
    ref = acc.reshape(Z, M, K).to(torch.complex128) @ site
    got = out.reshape(Z, M, N).to(torch.complex128)
    err = ((got - ref).norm() / ref.norm()).item()
    assert err <= 6e-6, err
    shrink = (torch.sum(got * ref.conj()).real / torch.sum(ref * ref.conj()).real).item() - 1.0
    assert abs(shrink) <= 5e-7, shrink
    want = torch.view_as_real(out.reshape(Z, -1)).abs().reshape(Z, -1).amax(dim=1)
    assert torch.equal(amax_out, want), (amax_out, want)


@pytest.mark.parametrize("dtype", ["complex64", "complex128"])
@pytest.mark.parametrize("M,K,N", [(65536, 16, 1), (65536, 8, 4), (65536, 2, 2), (65536, 64, 3), (131072, 32, 2), (65536, 8, 16), (65536, 4, 8), (65536, 2, 16), (65536, 16, 12),
                                   (4, 16, 2048), (32, 2048, 16), (1, 512, 2), (1, 8192, 16), (256, 8192, 16),
                                   # split-K: few rows, long K
                                   (1024, 32768, 64), (341, 4096, 64), (1, 65536, 32)])
def test_skinny_and_few_row_steps(M, K, N, dtype):
    """Warp-cooperative skinny kernel (complex64, K <= 64, N <= 4) and the
    few-row kernel (Z*M < 4096) against the complex128 product of the same
    operands, through tnc_step with automatic kernel choice."""
    import ctypes as C

    import torch

    from paper_2011_02621_b200 import _native as NV
    from paper_2011_02621_b200.engine import ContractionPlan, NetworkSpec, PathExecutor

    edges = {(0, 1): K, (0, 2): M, (1, 2): N}
    legs = {0: [(0, 2), (0, 1)], 1: [(0, 1), (1, 2)], 2: [(0, 2), (1, 2)]}
    spec = NetworkSpec([0, 1, 2], edges, legs)
    tdt = getattr(torch, dtype)
    g = torch.Generator(device="cuda")
    g.manual_seed(M * 7 + K * 3 + N)
    sites = {q: torch.randn((1,) + spec.site_dims(q), dtype=tdt, device="cuda", generator=g) for q in range(3)}
    plan = ContractionPlan(spec, [0, 1, 2])
    sp = plan.steps[0]
    assert (sp.M, sp.K, sp.N) == (M, K, N)
    ex = PathExecutor(plan, sites, dtype=dtype)
    d = ex._steps[0]
    Z = 3
    acc = torch.randn(Z * M * K, dtype=tdt, device="cuda", generator=g)
    out = torch.zeros(Z * M * N, dtype=tdt, device="cuda")
    d.Z, d.slices_per_b, d.s0 = Z, 1, 0
    d.acc, d.acc_zstride = acc.data_ptr(), M * K
    d.out, d.out_zstride = out.data_ptr(), M * N
    d.site.sel = None
    d.amax_in = d.amax_out = None
    NV.check(NV.lib().tnc_step(C.byref(d), C.c_void_p(torch.cuda.current_stream().cuda_stream)), "tnc_step")
    torch.cuda.synchronize()
    site = ex.step_sites[0][0][0].reshape(K, N).to(torch.complex128)
    ref = acc.reshape(Z, M, K).to(torch.complex128) @ site
    err = ((out.reshape(Z, M, N).to(torch.complex128) - ref).norm() / ref.norm()).item()
    assert err <= (2e-6 if dtype == "complex64" else 1e-13), err
