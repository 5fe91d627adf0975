"""GPU parity: the sm_100a engine (through the libtnc C ABI) against the
reference's golden amplitudes and the CPU oracle.

Tolerances (north star): relative L2 over a batch <= 1e-10 in complex128 and
<= 1e-4 in complex64; contraction paths / slice plans bit-exact.
"""

import json

import numpy as np
import pytest

import tn_oracle as O
from conftest import GOLDEN

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _device():
    import torch

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2011_02621_b200 import _native

    _native.require_device()
    torch.cuda.set_device(0)


def rel_l2(got, ref):
    ref = np.asarray(ref)
    return float(np.linalg.norm(np.asarray(got) - ref) / max(np.linalg.norm(ref), 1e-300))


def test_contract_pair_matches_reference_golden():
    from paper_2011_02621_b200 import Tensor, contract_pair

    meta = json.loads((GOLDEN / "pairs.json").read_text())
    arr = np.load(GOLDEN / "pairs.npz")
    for t, m in enumerate(meta["pairs"]):
        a = Tensor(arr[f"a{t}"], tuple(f"a{i}" for i in range(arr[f"a{t}"].ndim)))
        b = Tensor(arr[f"b{t}"], tuple(f"b{i}" for i in range(arr[f"b{t}"].ndim)))
        out = contract_pair(a, b, [tuple(p) for p in m["pairs"]])
        np.testing.assert_allclose(out.data, arr[f"out{t}"], atol=1e-12)


def test_compute_amplitude_matches_reference(golden_amplitudes):
    """Single-amplitude drop-in (reference default split / cuts / rank cap)."""
    from paper_2011_02621_b200 import compute_amplitude, parse_circuit

    worst = 0.0
    for case in golden_amplitudes:
        c = parse_circuit(case["circuit"])
        cuts = [tuple(e) for e in case["cuts"]] if isinstance(case["cuts"], list) else case["cuts"]
        for r in case["results"][:3]:
            st = compute_amplitude(c, case["in_bits"], r["out"], split_cycle=case["split_cycle"],
                                   cuts=cuts, max_rank=case["max_rank"])
            worst = max(worst, abs(st.amplitude - complex(*r["amplitude"])))
            assert st.path == r["path"] and str(st.path_score) == r["path_score"]
            assert st.slice_count == r["slice_count"] and st.peak_rank == r["peak_rank"]
            assert str(st.multiplies) == r["multiplies"]
    assert worst <= 1e-10


@pytest.mark.parametrize("dtype,tol", [("complex128", 1e-10), ("complex64", 1e-4)])
def test_projected_batch_config0(golden_amplitudes, dtype, tol):
    """BASELINE configs[0]: 3x3, 8 cycles, 64 bitstrings, batched gather path."""
    from paper_2011_02621_b200 import AmplitudeEngine, parse_circuit

    case = golden_amplitudes[0]
    c = parse_circuit(case["circuit"])
    eng = AmplitudeEngine(c, case["in_bits"], dtype=dtype)
    assert eng.path == case["results"][0]["path"]
    outs = [r["out"] for r in case["results"]]
    got = eng.amplitudes(outs)
    ref = np.array([complex(*r["amplitude"]) for r in case["results"]])
    assert rel_l2(got, ref) <= tol
    sv = np.array([complex(*r["statevector"]) for r in case["results"]])
    assert rel_l2(got, sv) <= tol


def test_two_sided_batch(golden_amplitudes):
    from paper_2011_02621_b200 import compute_amplitudes, parse_circuit

    case = golden_amplitudes[1]
    c = parse_circuit(case["circuit"])
    outs = [r["out"] for r in case["results"]]
    res = compute_amplitudes(c, case["in_bits"], outs, split_cycle=c.depth // 2, cuts="auto")
    ref = np.array([complex(*r["amplitude"]) for r in case["results"]])
    assert rel_l2(res.amplitudes, ref) <= 1e-10


@pytest.mark.parametrize("dtype,tol", [("complex128", 1e-10), ("complex64", 1e-4)])
def test_projected_with_cuts_slice_sum(golden_amplitudes, dtype, tol):
    """Cut plans: all slices x all bitstrings in one batched pass, summed."""
    from paper_2011_02621_b200 import AmplitudeEngine, parse_circuit

    case = golden_amplitudes[0]
    c = parse_circuit(case["circuit"])
    outs = [r["out"] for r in case["results"]][:32]
    ref = np.array([complex(*r["statevector"]) for r in case["results"]][:32])
    for cuts in ([(0, 1)], [(1, 4), (4, 5)], [(0, 3), (4, 7), (5, 8)]):
        eng = AmplitudeEngine(c, case["in_bits"], cuts=cuts, dtype=dtype)
        assert eng.cut_plan.slice_count > 1
        got = eng.amplitudes(outs)
        assert rel_l2(got, ref) <= tol, cuts
        # chunked over slices (forced small batch) gives the same sums
        eng2 = AmplitudeEngine(c, case["in_bits"], cuts=cuts, dtype=dtype, max_batch_elems=3)
        got2 = eng2.amplitudes(outs)
        assert rel_l2(got2, ref) <= tol


def test_projected_larger_lattice(golden_amplitudes):
    from paper_2011_02621_b200 import AmplitudeEngine, parse_circuit

    case = golden_amplitudes[-1]   # 5x4, 6 cycles, split = depth
    c = parse_circuit(case["circuit"])
    outs = [r["out"] for r in case["results"]]
    ref = np.array([complex(*r["amplitude"]) for r in case["results"]])
    eng = AmplitudeEngine(c, case["in_bits"], dtype="complex128")
    assert eng.path == case["results"][0]["path"]
    assert rel_l2(eng.amplitudes(outs), ref) <= 1e-10


def test_build_overlap_network_and_contract_along_path(golden_amplitudes):
    from paper_2011_02621_b200 import (build_overlap_network, contract_along_path,
                                       fuse_single_qubit_gates, parse_circuit, two_sided_evolve)

    case = golden_amplitudes[3]
    c = parse_circuit(case["circuit"])
    r = case["results"][0]
    fused = fuse_single_qubit_gates(c)
    phi, psi = two_sided_evolve(fused, case["in_bits"], r["out"], case["split_cycle"])
    net = build_overlap_network(phi, psi)
    n = c.num_qubits
    ne = {q: c.graph.node_edges(q) for q in range(n)}
    ref = O.overlap_tensors({q: (phi.tensors[q].data, list(phi.tensors[q].labels)) for q in range(n)},
                            {q: (psi.tensors[q].data, list(psi.tensors[q].labels)) for q in range(n)},
                            ne, phi.bond_dims, psi.bond_dims)
    for q in range(n):
        np.testing.assert_allclose(net.tensors[q].data, ref[q][0], atol=1e-13)
    val, stats = contract_along_path(net, sorted(net.tensors))
    want, peak, mult = O.contract_along_path(ref, sorted(net.tensors))
    assert abs(val - want) < 1e-12 and stats["peak_rank"] == peak and stats["multiplies"] == mult


def _sweep_case(rng, r, k, n, B, dtype):
    import torch

    legs = list(range(r + k))
    perm = list(rng.permutation(legs))
    dims = [2 if x < r else 4 for x in perm]
    size = int(np.prod(dims))
    acc = (rng.standard_normal((B, size)) + 1j * rng.standard_normal((B, size))) / np.sqrt(2)
    site = (rng.standard_normal((2, 4 ** k, 4 ** n)) + 1j * rng.standard_normal((2, 4 ** k, 4 ** n))) / 2
    bits = rng.integers(0, 2, B)
    return perm, dims, acc, site.reshape((2,) + (4,) * (k + n)), bits


@pytest.mark.parametrize("r,k,n,B", [(10, 1, 1, 4), (9, 2, 1, 3), (8, 3, 1, 2), (8, 1, 3, 2), (7, 2, 2, 5),
                                     (7, 3, 3, 2), (12, 2, 3, 1), (6, 3, 2, 8)])
@pytest.mark.parametrize("dtype,tol", [("complex128", 1e-12), ("complex64", 1e-5)])
def test_sweep_step_matches_oracle(r, k, n, B, dtype, tol):
    """BASELINE configs[1] at test sizes: permuted accumulator legs, projected
    site per bitstring, the fused permute+contract kernel vs the oracle."""
    import torch

    from paper_2011_02621_b200.engine import contract_pair_device

    rng = np.random.default_rng(r * 100 + k * 10 + n)
    perm, dims, acc, site, bits = _sweep_case(rng, r, k, n, B, dtype)
    tdt = torch.complex64 if dtype == "complex64" else torch.complex128
    ta = torch.from_numpy(acc).to("cuda", tdt)
    sites_b = site[bits].reshape(B, -1)
    tb = torch.from_numpy(np.ascontiguousarray(sites_b)).to("cuda", tdt)
    shared_pos = sorted((i for i, x in enumerate(perm) if x >= r), key=lambda i: perm[i])
    pairs = [(p, j) for j, p in enumerate(shared_pos)]
    out = contract_pair_device(ta, dims, tb, [4] * (k + n), pairs, batch=B,
                               a_zstride=acc.shape[1], b_zstride=sites_b.shape[1])
    got = out.cpu().numpy().astype(np.complex128)
    ref = O.sweep_step(acc, perm, r, k, site, bits)
    assert rel_l2(got, ref) <= tol


@pytest.mark.parametrize("r,kdims,ndims", [(15, (4,), (4, 4)), (15, (2, 2), (4, 2, 2)), (13, (4,), (4, 4, 4)),
                                           (12, (4, 4), (4, 4)), (9, (4,), (4, 4)), (6, (4,), (4, 4))])
def test_pipe_cols_variant(r, kdims, ndims):
    """complex64, K <= 16, 16 <= N <= 64: the column-mapped k_pair_pipe_cols
    (two columns per thread) on permuted accumulators, many tiles per CTA and
    several z, against tensordot"""
    import torch

    from paper_2011_02621_b200.engine import contract_pair_device

    rng = np.random.default_rng(r + 7 * len(ndims))
    B = 3
    legs = [2] * r + list(kdims)
    perm = list(rng.permutation(len(legs)))
    a_dims = [legs[x] for x in perm]
    shared_pos = [perm.index(r + j) for j in range(len(kdims))]
    b_dims = list(kdims) + list(ndims)
    pairs = [(shared_pos[j], j) for j in range(len(kdims))]
    acc = (rng.standard_normal((B,) + tuple(a_dims)) + 1j * rng.standard_normal((B,) + tuple(a_dims))).astype(np.complex64)
    site = (rng.standard_normal((B,) + tuple(b_dims)) + 1j * rng.standard_normal((B,) + tuple(b_dims))).astype(np.complex64)
    ta = torch.from_numpy(acc.reshape(B, -1)).cuda()
    tb = torch.from_numpy(site.reshape(B, -1)).cuda()
    out = contract_pair_device(ta, a_dims, tb, b_dims, pairs, batch=B, a_zstride=ta.shape[1], b_zstride=tb.shape[1])
    got = out.cpu().numpy().astype(np.complex128)
    ref = np.stack([np.tensordot(acc[z].astype(np.complex128), site[z].astype(np.complex128),
                                 axes=(shared_pos, list(range(len(kdims))))).reshape(-1) for z in range(B)])
    assert rel_l2(got, ref) <= 1e-5


@pytest.mark.parametrize("kdims,ndims", [((4, 4), ()), ((4, 4), (2,)), ((4, 4), (4,)), ((2, 4), (4,)),
                                         ((4, 2, 2), (2, 2))])
@pytest.mark.parametrize("dtype,tol", [("complex128", 1e-12), ("complex64", 1e-5)])
def test_pipe_producer_variant(kdims, ndims, dtype, tol):
    """K >= 8, N <= 4: the producer-warp k_pair_pipe (mbarrier stage release)
    on a permuted accumulator with many tiles per CTA, against tensordot."""
    import torch

    from paper_2011_02621_b200.engine import contract_pair_device

    rng = np.random.default_rng(len(kdims) * 10 + len(ndims))
    r, B = 15, 3
    legs = [2] * r + list(kdims)
    perm = list(rng.permutation(len(legs)))
    a_dims = [legs[x] for x in perm]
    shared_pos = [perm.index(r + j) for j in range(len(kdims))]
    b_dims = list(kdims) + list(ndims)
    pairs = [(shared_pos[j], j) for j in range(len(kdims))]
    cdt = np.complex64 if dtype == "complex64" else np.complex128
    acc = (rng.standard_normal((B,) + tuple(a_dims)) + 1j * rng.standard_normal((B,) + tuple(a_dims))).astype(cdt)
    site = (rng.standard_normal((B,) + tuple(b_dims)) + 1j * rng.standard_normal((B,) + tuple(b_dims))).astype(cdt)
    tdt = torch.complex64 if dtype == "complex64" else torch.complex128
    ta = torch.from_numpy(acc.reshape(B, -1)).to("cuda", tdt)
    tb = torch.from_numpy(site.reshape(B, -1)).to("cuda", tdt)
    out = contract_pair_device(ta, a_dims, tb, b_dims, pairs, batch=B, a_zstride=ta.shape[1], b_zstride=tb.shape[1])
    got = out.cpu().numpy().astype(np.complex128)
    ref = np.stack([np.tensordot(acc[z].astype(np.complex128), site[z].astype(np.complex128),
                                 axes=(shared_pos, list(range(len(kdims))))).reshape(-1) for z in range(B)])
    assert rel_l2(got, ref) <= tol


def test_kernel_variants_agree(golden_amplitudes):
    """Forcing the generic kernel gives the same amplitudes as the tuned path."""
    from paper_2011_02621_b200 import AmplitudeEngine, parse_circuit
    from paper_2011_02621_b200 import _native as NV

    case = golden_amplitudes[0]
    c = parse_circuit(case["circuit"])
    outs = [r["out"] for r in case["results"]][:16]
    eng = AmplitudeEngine(c, case["in_bits"], dtype="complex128")
    base = eng.amplitudes(outs)
    for i in range(len(eng.plan.steps)):
        eng.executor._steps[i].kernel = NV.K_GENERIC
    forced = eng.amplitudes(outs)
    np.testing.assert_allclose(forced, base, atol=1e-13)


def test_linearity_and_slice_identity_at_scale():
    """Size-independent properties on a 53-qubit Sycamore-style network
    (8 cycles): scaling one site tensor scales every amplitude; a cut plan's
    slice sum equals the uncut contraction."""
    import torch

    from paper_2011_02621_b200 import AmplitudeEngine, pattern_rqc, sycamore53_graph

    graph, pats, _ = sycamore53_graph()
    seq = [pats[ch] for ch in "ABCDCDAB"]
    c = pattern_rqc(graph, seq, 4, seed=3)
    rng = np.random.default_rng(5)
    outs = ["".join(rng.choice(["0", "1"], 53)) for _ in range(8)]
    eng = AmplitudeEngine(c, dtype="complex128", max_rank=10)
    base = eng.amplitudes(outs)
    assert np.all(np.isfinite(base)) and np.linalg.norm(base) > 0
    # linearity in one site tensor
    q = eng.path[len(eng.path) // 2]
    eng2 = AmplitudeEngine(c, dtype="complex128", max_rank=10)
    eng2.executor.raw[q].mul_(2.5 - 1.0j)
    eng2.executor.__init__(eng2.plan, {p: eng2.executor.raw[p] for p in eng2.plan.spec.nodes}, dtype="complex128")
    scaled = eng2.amplitudes(outs)
    np.testing.assert_allclose(scaled, (2.5 - 1.0j) * base, rtol=1e-10, atol=1e-300)
    # slice identity: cut two edges on the path's frontier
    e1, e2 = sorted(eng.edges)[10], sorted(eng.edges)[40]
    eng3 = AmplitudeEngine(c, dtype="complex128", max_rank=10, cuts=[e1, e2])
    assert rel_l2(eng3.amplitudes(outs), base) <= 1e-10


def test_sharded_ranks_sum_to_full(golden_amplitudes):
    """Two ranks' shards (simulated in one process) of a sliced batch sum to
    the single-pass amplitudes: b_offset / slice-range execution is exact."""
    import torch

    from paper_2011_02621_b200 import AmplitudeEngine, parse_circuit
    from paper_2011_02621_b200.distributed import run_sharded

    case = golden_amplitudes[0]
    c = parse_circuit(case["circuit"])
    outs = [r["out"] for r in case["results"]][:5]
    ref = np.array([complex(*r["statevector"]) for r in case["results"]][:5])
    eng = AmplitudeEngine(c, case["in_bits"], cuts=[(1, 4), (4, 5)], dtype="complex128")
    bits = np.array([[int(ch) for ch in b] for b in outs], dtype=np.int32)
    sel = eng.selectors(bits)
    total = torch.zeros(5, dtype=torch.complex128, device="cuda")
    for world in (2, 3, 8):
        total.zero_()
        for rank in range(world):
            part = torch.zeros(5, dtype=torch.complex128, device="cuda")
            run_sharded(eng.executor, sel, 5, part, rank, world)
            total += part
        assert rel_l2(total.cpu().numpy(), ref) <= 1e-12


def test_graph_replay_matches_eager(golden_amplitudes):
    """CUDA-graph replay of whole path chunks gives the eager amplitudes, also
    after the inputs change in place (same buffers, new bitstrings)."""
    import torch

    from paper_2011_02621_b200 import AmplitudeEngine, parse_circuit

    case = golden_amplitudes[0]
    c = parse_circuit(case["circuit"])
    outs = [r["out"] for r in case["results"]][:16]
    eng = AmplitudeEngine(c, case["in_bits"], dtype="complex128")
    nq = c.num_qubits
    bits = np.array([[int(ch) for ch in o] for o in outs], dtype=np.int32)
    sel = eng.selectors(bits)
    base = eng.amplitudes_device(sel, len(outs)).cpu().numpy()
    amp = torch.zeros(len(outs), dtype=torch.complex128, device="cuda")
    for _ in range(3):                     # eager, capture, replay
        eng.amplitudes_device(sel, len(outs), amp, graph=True)
    np.testing.assert_allclose(amp.cpu().numpy(), base, atol=1e-13)
    flipped = 1 - bits
    sel2 = eng.selectors(flipped)
    for q in sel:                          # same device buffers, new contents
        if sel[q] is not None:
            sel[q].copy_(sel2[q])
    eng.amplitudes_device(sel, len(outs), amp, graph=True)
    ref = eng.amplitudes(["".join(map(str, row)) for row in flipped])
    np.testing.assert_allclose(amp.cpu().numpy(), ref, atol=1e-13)
    assert nq == bits.shape[1]


def test_sycamore53_sliced_matches_unsliced():
    """53-qubit Sycamore (ABCDCDAB, 8 cycles): the projected engine sliced over
    the bench's depth-10 cut edges (network.py:173-243 scheme: cut legs fixed
    per slice, device slice sum) against the unsliced network, complex64."""
    from paper_2011_02621_b200 import AmplitudeEngine, pattern_rqc, sycamore53_graph

    graph, pats, _ = sycamore53_graph()
    circ = pattern_rqc(graph, [pats[c] for c in "ABCDCDAB"], 8, seed=0)
    rng = np.random.default_rng(11)
    outs = ["".join(map(str, r)) for r in rng.integers(0, 2, (2, 53))]
    ref = AmplitudeEngine(circ, dtype="complex64", max_rank=12).amplitudes(outs, graph=False)
    eng = AmplitudeEngine(circ, dtype="complex64", max_rank=12, cuts=[(9, 14), (2, 9)])
    assert eng.plan.slice_count > 1
    got = eng.amplitudes(outs, graph=False)
    assert rel_l2(got, ref) <= 1e-4
