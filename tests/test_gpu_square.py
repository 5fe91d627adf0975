"""GPU parity on the square-lattice configs of BASELINE.json.

configs[2] (5x4, 20 qubits): two-sided amplitudes against the dense 2^20 state
vector (oracle ``statevector_amplitudes``, the reference's oracle.py:68-96) at
14 cycles unsliced (2^31-element intermediates, 3.7e13 multiplies per
amplitude) in complex64 and complex128, and at 12 cycles through the cut edges
(4,8), (11,15) of the 16-cycle plan (tools/full_amplitude.py runs the 16-cycle
amplitude itself: 16384 slices, about 1.6 GPU hours, profiles/).

configs[3] (7x7, 49 qubits): against amplitudes computed by the REFERENCE
(tests/golden/square.json, tests/golden/make_golden_square.py) at 8 cycles with
the reference's default rank cap M = treewidth bound + 1, unsliced and with
explicit cut edges; path, score, peak rank, multiplies and slice count
bit-exact.
"""

import json

import numpy as np
import pytest

import tn_oracle as O
from conftest import GOLDEN

pytestmark = pytest.mark.gpu

TOL = {"complex128": 1e-10, "complex64": 1e-4}


@pytest.fixture(scope="module", autouse=True)
def _device():
    import torch

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2011_02621_b200 import _native

    _native.require_device()
    torch.cuda.set_device(0)


def rel_l2(got, ref):
    ref = np.asarray(ref)
    return float(np.linalg.norm(np.asarray(got) - ref) / np.linalg.norm(ref))


def _square(rows, cols, depth, seed=0):
    from paper_2011_02621_b200 import generate_lattice, pattern_rqc, square_patterns

    g = generate_lattice("square", rows, cols)
    return pattern_rqc(g, square_patterns(rows, cols), depth, seed=seed)


@pytest.mark.parametrize("dtype,nbits", [("complex64", 8), ("complex128", 2)])
def test_cfg2_5x4_d14_matches_statevector(dtype, nbits):
    """configs[2] circuit at 14 cycles: whole two-sided amplitudes (split 7,
    intermediates up to 2^31 elements) vs the dense state vector."""
    import torch

    from paper_2011_02621_b200.network import TwoSidedEngine

    circ = _square(5, 4, 14)
    rng = np.random.default_rng(14)
    outs = ["".join(rng.choice(["0", "1"], 20)) for _ in range(nbits)]
    ref = O.statevector_amplitudes(circ, "0" * 20, outs)
    eng = TwoSidedEngine(circ, split_cycle=7, cuts=None, max_rank=6, dtype=dtype, max_batch_elems=1)
    assert eng.plan.max_elems == 1 << 31 and eng.plan.slice_count == 1
    got = eng.amplitudes(outs)
    torch.cuda.synchronize()
    err = rel_l2(got, ref)
    assert err <= TOL[dtype], f"5x4 d14 {dtype}: rel L2 {err:.3e}"


@pytest.mark.parametrize("dtype", ["complex64", "complex128"])
def test_cfg2_5x4_d12_sliced_matches_statevector(dtype):
    """The slicing scheme of the 16-cycle plan (cut edges (4,8), (11,15)) at 12
    cycles: 1024 slices summed on the device vs the dense state vector."""
    from paper_2011_02621_b200.network import TwoSidedEngine

    circ = _square(5, 4, 12)
    rng = np.random.default_rng(12)
    outs = ["".join(rng.choice(["0", "1"], 20)) for _ in range(4)]
    ref = O.statevector_amplitudes(circ, "0" * 20, outs)
    eng = TwoSidedEngine(circ, split_cycle=6, cuts=[(4, 8), (11, 15)], max_rank=6, dtype=dtype)
    assert eng.plan.slice_count == 1024
    got = eng.amplitudes(outs)
    # the slice sum cancels: complex64 keeps 1e-4 of the amplitude norm, not of each slice
    err = rel_l2(got, ref)
    assert err <= (2e-4 if dtype == "complex64" else 1e-10), f"5x4 d12 sliced {dtype}: rel L2 {err:.3e}"
    # slice ranges add up (the multi-GPU split)
    part = sum(eng.amplitudes(outs, slices=range(lo, lo + 256)) for lo in range(0, 1024, 256))
    assert rel_l2(part, got) <= (2e-4 if dtype == "complex64" else 1e-10)


def _cfg3_cases():
    return json.loads((GOLDEN / "square.json").read_text())["cases"]


@pytest.mark.parametrize("dtype", ["complex128", "complex64"])
@pytest.mark.parametrize("name", [c["name"] for c in json.loads((GOLDEN / "square.json").read_text())["cases"]])
def test_cfg3_7x7_matches_reference(name, dtype):
    from paper_2011_02621_b200 import parse_circuit
    from paper_2011_02621_b200.network import TwoSidedEngine

    case = next(c for c in _cfg3_cases() if c["name"] == name)
    c = parse_circuit(case["circuit"])
    cuts = [tuple(e) for e in case["cuts"]] if case["cuts"] else None
    eng = TwoSidedEngine(c, case["in_bits"], split_cycle=case["split_cycle"], cuts=cuts,
                         max_rank=case["max_rank"], dtype=dtype)
    r0 = case["results"][0]
    assert eng.path == r0["path"]
    assert str(eng.path_score) == r0["path_score"]
    assert eng.plan.peak_rank == r0["peak_rank"]
    assert str(eng.plan.multiplies) == r0["multiplies"]
    assert eng.cut_plan.slice_count == r0["slice_count"]
    outs = [r["out"] for r in case["results"]]
    got = eng.amplitudes(outs)
    ref = np.array([complex(*r["amplitude"]) for r in case["results"]])
    err = rel_l2(got, ref)
    assert err <= TOL[dtype], f"{name} {dtype}: rel L2 {err:.3e}"
