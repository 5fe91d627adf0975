"""GPU parity on the 53-qubit Sycamore family (BASELINE configs[4]) against
amplitudes computed by the REFERENCE itself (tests/golden/syc53.json, written
by tests/golden/make_golden_syc53.py with tnsim.compute_amplitude).

Covers both network forms the bench reports -- projected (split = depth,
``AmplitudeEngine``) and two-sided (split = depth // 2, ``TwoSidedEngine``,
the reference default) -- unsliced and with explicit cut plans (the bench's
slicing scheme), in complex128 (rel L2 <= 1e-10) and complex64 (<= 1e-4), with
path, path score, peak rank, multiplies and slice count bit-exact.
"""

import json

import numpy as np
import pytest

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


def _cases():
    return json.loads((GOLDEN / "syc53.json").read_text())["cases"]


def rel_l2(got, ref):
    ref = np.asarray(ref)
    return float(np.linalg.norm(np.asarray(got) - ref) / np.linalg.norm(ref))


def _engine(case, dtype):
    from paper_2011_02621_b200 import AmplitudeEngine, parse_circuit
    from paper_2011_02621_b200.network import TwoSidedEngine

    c = parse_circuit(case["circuit"])
    cuts = [tuple(e) for e in case["cuts"]] if case["cuts"] else None
    if case["split_cycle"] == c.depth:
        return AmplitudeEngine(c, case["in_bits"], cuts=cuts, max_rank=case["max_rank"], dtype=dtype)
    return TwoSidedEngine(c, case["in_bits"], split_cycle=case["split_cycle"], cuts=cuts,
                          max_rank=case["max_rank"], dtype=dtype)


@pytest.mark.parametrize("dtype", ["complex128", "complex64"])
@pytest.mark.parametrize("name", [c["name"] for c in json.loads((GOLDEN / "syc53.json").read_text())["cases"]])
def test_syc53_matches_reference(name, dtype):
    case = next(c for c in _cases() if c["name"] == name)
    eng = _engine(case, dtype)
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


def test_syc53_compute_amplitude_drop_in():
    """The single-amplitude drop-in on a two-sided 53-qubit golden (c128)."""
    from paper_2011_02621_b200 import compute_amplitude, parse_circuit

    case = next(c for c in _cases() if c["name"] == "syc53_d8_twosided")
    c = parse_circuit(case["circuit"])
    r = case["results"][0]
    st = compute_amplitude(c, case["in_bits"], r["out"], split_cycle=case["split_cycle"], cuts=None,
                           max_rank=case["max_rank"])
    assert st.path == r["path"] and str(st.path_score) == r["path_score"]
    assert abs(st.amplitude - complex(*r["amplitude"])) <= 1e-10 * abs(complex(*r["amplitude"]))


def test_two_sided_engine_batches_and_slice_ranges():
    """One executor reloaded with different bitstring batches gives the same
    amplitudes as fresh engines, and slice ranges sum to the full amplitude."""
    case = next(c for c in _cases() if c["name"] == "syc53_d8_twosided_cut")
    eng = _engine(case, "complex128")
    outs = [r["out"] for r in case["results"]]
    ref = np.array([complex(*r["amplitude"]) for r in case["results"]])
    S = eng.cut_plan.slice_count
    for _ in range(2):                                   # second round reloads the same executor
        for b in range(len(outs)):
            got = eng.amplitudes([outs[b]])
            assert abs(got[0] - ref[b]) <= 1e-10 * abs(ref[b])
    part = sum(eng.amplitudes(outs, slices=range(lo, min(lo + 300, S))) for lo in range(0, S, 300))
    assert rel_l2(part, ref) <= 1e-10
