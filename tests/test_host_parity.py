"""Host-side parity with the reference (CPU only).

Golden fixtures come from the reference itself (tests/golden/make_golden.py).
Checks: circuits byte-identical, network shapes identical, contraction path /
score / slice plan / peak rank / multiply count bit-exact, the CPU oracle
reproduces the reference amplitudes, and the engine's device descriptors
(interpreted in numpy) reproduce the oracle.
"""

import json

import numpy as np
import pytest

import tn_oracle as O
from paper_2011_02621_b200 import (find_optimal_path, fuse_single_qubit_gates, parse_circuit,
                                   serialize_circuit, treewidth_bound, two_sided_evolve)
from paper_2011_02621_b200.engine import ContractionPlan, NetworkSpec
from paper_2011_02621_b200.network import _ShapeNet, _path_for, _resolve_cuts, plan_cuts
from paper_2011_02621_b200.pathfind import NetworkShape, PathSearchError, exhaustive_path_oracle
from plan_interp import run_plan

from conftest import GOLDEN


def _cuts(spec):
    return [tuple(e) for e in spec] if isinstance(spec, list) else spec


def _case_network(case, out_bits):
    c = parse_circuit(case["circuit"])
    fused = fuse_single_qubit_gates(c)
    phi, psi = two_sided_evolve(fused, case["in_bits"], out_bits, case["split_cycle"])
    edges = {e: phi.bond_dims[e] * psi.bond_dims[e] for e in c.graph.edges}
    return c, phi, psi, edges


def test_circuits_serialize_byte_identical(golden_amplitudes):
    for case in golden_amplitudes:
        assert serialize_circuit(parse_circuit(case["circuit"])).decode() == case["circuit"]


def test_network_shape_path_and_plan_bit_exact(golden_amplitudes):
    checked = 0
    for case in golden_amplitudes:
        for r in case["results"]:
            c, phi, psi, edges = _case_network(case, r["out"])
            if r is case["results"][0]:
                assert edges == {(k, l): x for k, l, x in case["edges"]}, case["name"]
            n = c.num_qubits
            sn = _ShapeNet(range(n), edges)
            plan = _resolve_cuts(sn, _cuts(case["cuts"]), case["max_rank"])
            path, score = _path_for(sn, plan, case["max_rank"])
            assert path == r["path"], case["name"]
            assert str(score) == r["path_score"], case["name"]
            assert plan.slice_count == r["slice_count"], case["name"]
            spec = NetworkSpec(list(range(n)), edges, {q: c.graph.node_edges(q) for q in range(n)})
            cp = ContractionPlan(spec, path, plan.cut_edges)
            assert cp.peak_rank == r["peak_rank"], case["name"]
            assert str(cp.multiplies) == r["multiplies"], case["name"]
            checked += 1
    assert checked >= 100


def test_oracle_reproduces_reference_amplitudes(golden_amplitudes):
    """Pins the CPU oracle: reference compute_amplitude values, to 1e-13."""
    worst = 0.0
    for case in golden_amplitudes:
        for r in case["results"][:8]:
            c, phi, psi, edges = _case_network(case, r["out"])
            n = c.num_qubits
            ne = {q: c.graph.node_edges(q) for q in range(n)}
            tens = O.overlap_tensors({q: (phi.tensors[q].data, list(phi.tensors[q].labels)) for q in range(n)},
                                     {q: (psi.tensors[q].data, list(psi.tensors[q].labels)) for q in range(n)},
                                     ne, phi.bond_dims, psi.bond_dims)
            sn = _ShapeNet(range(n), edges)
            plan = _resolve_cuts(sn, _cuts(case["cuts"]), case["max_rank"])
            amp = O.sliced_amplitude(tens, r["path"], plan.cut_edges, plan.extents)
            worst = max(worst, abs(amp - complex(*r["amplitude"])))
    assert worst <= 1e-13


def test_statevector_oracle_matches_reference(golden_amplitudes):
    for case in golden_amplitudes:
        c = parse_circuit(case["circuit"])
        outs = [r["out"] for r in case["results"]]
        got = O.statevector_amplitudes(c, case["in_bits"], outs)
        ref = np.array([complex(*r["statevector"]) for r in case["results"]])
        np.testing.assert_allclose(got, ref, atol=1e-14)


def test_tns_amplitudes_match_statevector(golden_amplitudes):
    """The reference's TNS amplitude equals the dense state vector (1e-10)."""
    for case in golden_amplitudes:
        for r in case["results"]:
            assert abs(complex(*r["amplitude"]) - complex(*r["statevector"])) <= 1e-10


def test_random_shape_paths_bit_exact(golden_paths):
    for rec in golden_paths["random"]:
        shape = NetworkShape(tuple(range(rec["n"])), {(k, l): x for k, l, x in rec["edges"]})
        for run in rec["runs"]:
            opts = dict(run["opts"])
            if "error" in run:
                with pytest.raises(PathSearchError) as exc:
                    find_optimal_path(shape, **opts)
                assert exc.value.largest_subset == run["largest"]
                assert str(exc.value) == run["error"]
            else:
                p, s = find_optimal_path(shape, **opts)
                assert p == run["path"] and str(s) == run["score"]
        if "exhaustive" in rec:
            p, s = exhaustive_path_oracle(shape)
            assert p == rec["exhaustive"]["path"] and str(s) == rec["exhaustive"]["score"]
        assert treewidth_bound(shape) == rec["treewidth"]


def test_lattice_paths_bit_exact(golden_paths):
    """53-qubit Sycamore (d=8, 12) and 7x7 networks: same path and score."""
    for rec in golden_paths["lattice"]:
        edges = {(k, l): x for k, l, x in rec["edges"]}
        n = 1 + max(max(e) for e in edges)
        shape = NetworkShape(tuple(range(n)), edges)
        p, s = find_optimal_path(shape, rec["cap"])
        assert p == rec["path"] and str(s) == rec["score"], rec["name"]
        assert treewidth_bound(shape) == rec["treewidth"]


def test_plan_cuts_bit_exact(golden_paths):
    for rec in golden_paths["cuts"]:
        edges = {(k, l): x for k, l, x in rec["edges"]}
        n = 1 + max(max(e) for e in edges)
        net = _ShapeNet(range(n), edges)
        if "error" in rec:
            with pytest.raises(Exception):
                plan_cuts(net, rec["cap"])
            continue
        plan = plan_cuts(net, rec["cap"])
        assert [list(e) for e in plan.cut_edges] == rec["cut_edges"]
        assert plan.slice_count == rec["slice_count"]


def test_oracle_pairwise_and_slicing_golden():
    meta = json.loads((GOLDEN / "pairs.json").read_text())
    arr = np.load(GOLDEN / "pairs.npz")
    for t, m in enumerate(meta["pairs"]):
        a, b = arr[f"a{t}"], arr[f"b{t}"]
        la = [f"a{i}" for i in range(a.ndim)]
        lb = [f"b{i}" for i in range(b.ndim)]
        for pa, pb in m["pairs"]:
            lb[pb] = la[pa]
        out, _ = O.contract_pair(a, la, b, lb)
        np.testing.assert_allclose(out, arr[f"out{t}"], atol=1e-12)
    net = meta["net"]
    tensors = {int(q): (arr[f"net_node{q}"], [tuple(e) for e in labs]) for q, labs in net["labels"].items()}
    cuts = [tuple(e) for e in net["cut_edges"]]
    ext = {(k, l): x for k, l, x in net["edges"]}
    for s in range(net["slice_count"]):
        sl = O.slice_tensors(tensors, cuts, [ext[e] for e in cuts], s)
        for q, (t, _) in sl.items():
            np.testing.assert_array_equal(t, arr[f"slice{s}_node{q}"])
    whole = O.contract_along_path(tensors, sorted(tensors))[0]
    assert abs(whole - complex(*net["whole"])) < 1e-13
    total = O.sliced_amplitude(tensors, sorted(tensors), cuts, [ext[e] for e in cuts])
    assert abs(total - whole) < 1e-12


@pytest.mark.parametrize("case_idx", [0, 2, 3, 5, 9, 10])
def test_engine_descriptors_interpreted(golden_amplitudes, case_idx):
    """The planner's layouts/tables (as the kernels read them) reproduce the
    reference amplitudes when interpreted in numpy."""
    case = golden_amplitudes[case_idx]
    r = case["results"][0]
    c, phi, psi, edges = _case_network(case, r["out"])
    n = c.num_qubits
    ne = {q: c.graph.node_edges(q) for q in range(n)}
    tens = O.overlap_tensors({q: (phi.tensors[q].data, list(phi.tensors[q].labels)) for q in range(n)},
                             {q: (psi.tensors[q].data, list(psi.tensors[q].labels)) for q in range(n)},
                             ne, phi.bond_dims, psi.bond_dims)
    sn = _ShapeNet(range(n), edges)
    plan = _resolve_cuts(sn, _cuts(case["cuts"]), case["max_rank"])
    spec = NetworkSpec(list(range(n)), edges, ne)
    cp = ContractionPlan(spec, r["path"], plan.cut_edges)
    sites = {q: tens[q][0][None] for q in range(n)}
    amp = run_plan(cp, sites, None, 1)[0]
    assert abs(amp - complex(*r["amplitude"])) < 1e-12


def test_projected_mode_interpreted(golden_amplitudes):
    """Projected mode (split == depth): one plan, bit-selected site variants."""
    case = golden_amplitudes[0]
    assert case["split_cycle"] == 8
    c = parse_circuit(case["circuit"])
    fused = fuse_single_qubit_gates(c)
    from paper_2011_02621_b200.tns import evolve, init_state

    n = c.num_qubits
    phi = evolve(init_state(c.graph, case["in_bits"]), fused)
    edges = dict(phi.bond_dims)
    ne = {q: c.graph.node_edges(q) for q in range(n)}
    variants = {}
    for q in range(n):
        a = phi.tensors[q]
        v = np.transpose(a.data, [0] + [a.axis(e) for e in ne[q]])
        if q in fused.trailing:
            v = np.tensordot(fused.trailing[q], v, axes=([1], [0]))
        variants[q] = v
    r0 = case["results"][0]
    spec = NetworkSpec(list(range(n)), edges, ne)
    cp = ContractionPlan(spec, r0["path"], ())
    outs = [r["out"] for r in case["results"]][:16]
    bits = np.array([[int(ch) for ch in b] for b in outs], dtype=np.int32)
    sel = {q: bits[:, q] for q in range(n)}
    got = run_plan(cp, variants, sel, len(outs))
    ref = np.array([complex(*r["amplitude"]) for r in case["results"][:16]])
    np.testing.assert_allclose(got, ref, atol=1e-13)
    orc = O.projected_amplitudes(variants, ne, r0["path"], bits)
    np.testing.assert_allclose(orc, ref, atol=1e-13)
