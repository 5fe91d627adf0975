"""Host-side parity on the 53-qubit Sycamore family (CPU only).

Against tests/golden/syc53.json (reference ``compute_amplitude`` outputs):
network shape, path, score, cut plan, peak rank and multiply count are
bit-exact for every case; the CPU oracle reproduces the reference amplitudes
on the cheap cases.  The batched bra evolution (``tns.psi_batch``) is checked
against per-bitstring ``two_sided_evolve`` (bond dims, and amplitudes through
the dense state vector on a small lattice).
"""

import json

import numpy as np
import pytest

import tn_oracle as O
from conftest import GOLDEN
from paper_2011_02621_b200 import (fuse_single_qubit_gates, generate_lattice, parse_circuit, pattern_rqc,
                                   square_patterns, sycamore53_graph, two_sided_evolve)
from paper_2011_02621_b200.engine import ContractionPlan, NetworkSpec
from paper_2011_02621_b200.network import _path_for, _resolve_cuts, _ShapeNet
from paper_2011_02621_b200.tns import RankMismatch, evolve, init_state, psi_batch

CASES = json.loads((GOLDEN / "syc53.json").read_text())["cases"]


def _network(case, out_bits):
    c = parse_circuit(case["circuit"])
    fused = fuse_single_qubit_gates(c)
    phi, psi = two_sided_evolve(fused, case["in_bits"], out_bits, case["split_cycle"])
    edges = {e: phi.bond_dims[e] * psi.bond_dims[e] for e in c.graph.edges}
    return c, phi, psi, edges


@pytest.mark.parametrize("name", [c["name"] for c in CASES])
def test_syc53_plan_bit_exact(name):
    case = next(c for c in CASES if c["name"] == name)
    r = case["results"][0]
    c, phi, psi, edges = _network(case, r["out"])
    n = c.num_qubits
    sn = _ShapeNet(range(n), edges)
    cuts = [tuple(e) for e in case["cuts"]] if case["cuts"] else None
    plan = _resolve_cuts(sn, cuts, case["max_rank"])
    path, score = _path_for(sn, plan, case["max_rank"])
    assert path == r["path"] and str(score) == r["path_score"]
    cp = ContractionPlan(NetworkSpec(list(range(n)), edges, {q: c.graph.node_edges(q) for q in range(n)}),
                         path, plan.cut_edges)
    assert cp.peak_rank == r["peak_rank"]
    assert str(cp.multiplies) == r["multiplies"]
    assert cp.slice_count == r["slice_count"]


@pytest.mark.parametrize("name", ["syc53_d6_projected"])
def test_oracle_reproduces_syc53_reference(name):
    case = next(c for c in CASES if c["name"] == name)
    for r in case["results"]:
        c, phi, psi, edges = _network(case, r["out"])
        n = c.num_qubits
        ne = {q: c.graph.node_edges(q) for q in range(n)}
        tens = O.overlap_tensors({q: (phi.tensors[q].data, list(phi.tensors[q].labels)) for q in range(n)},
                                 {q: (psi.tensors[q].data, list(psi.tensors[q].labels)) for q in range(n)},
                                 ne, phi.bond_dims, psi.bond_dims)
        amp = O.sliced_amplitude(tens, r["path"])
        ref = complex(*r["amplitude"])
        assert abs(amp - ref) <= 1e-12 * abs(ref)


def test_psi_batch_matches_single_evolution_syc53():
    """Stacked-SVD batch evolution keeps the reference's bond dims per member."""
    graph, pats, _ = sycamore53_graph()
    circ = pattern_rqc(graph, [pats[ch] for ch in "ABCDCDAB"], 8, seed=0)
    fused = fuse_single_qubit_gates(circ)
    rng = np.random.default_rng(3)
    outs = ["".join(rng.choice(["0", "1"], 53)) for _ in range(6)]
    pb = psi_batch(fused, outs, 4)
    assert pb.batch == 6
    for o in outs[:2]:
        _, psi = two_sided_evolve(fused, "0" * 53, o, 4)
        assert psi.bond_dims == pb.bond_dims


def test_psi_batch_amplitudes_match_statevector():
    """<psi_b|phi> from the batched bras equals the dense state vector."""
    g = generate_lattice("square", 3, 4)
    circ = pattern_rqc(g, square_patterns(3, 4), 8, seed=3)
    fused = fuse_single_qubit_gates(circ)
    rng = np.random.default_rng(0)
    outs = ["".join(rng.choice(["0", "1"], 12)) for _ in range(8)]
    pb = psi_batch(fused, outs, 4)
    phi = evolve(init_state(fused.graph, "0" * 12), fused, range(0, 4), "forward")
    ref = O.statevector_amplitudes(circ, "0" * 12, outs)
    ne = {q: fused.graph.node_edges(q) for q in range(12)}
    path = list(range(12))
    for i in range(len(outs)):
        tens = O.overlap_tensors({q: (phi.tensors[q].data, list(phi.tensors[q].labels)) for q in range(12)},
                                 {q: (pb.tensors[q][i], ["p"] + list(ne[q])) for q in range(12)},
                                 ne, phi.bond_dims, pb.bond_dims)
        assert abs(O.sliced_amplitude(tens, path) - ref[i]) <= 1e-12


def test_psi_batch_rank_mismatch_detected():
    """Members whose compressions keep different ranks cannot share a pass."""
    from paper_2011_02621_b200.tns import TNSBatch, _compress_batch

    g = generate_lattice("square", 2, 2)
    e = (0, 1)
    assert g.node_edges(0)[0] == e and g.node_edges(1)[0] == e
    t0 = np.zeros((2, 2, 2, 1), dtype=np.complex128)     # [B, phys, bond (0,1), bond (0,2)]
    t0[0, :, :, 0] = np.eye(2)             # member 0: rank 2
    t0[1, :, 0, 0] = 1.0                   # member 1: rank 1
    t1 = np.ones((2, 2, 2, 1), dtype=np.complex128)
    st = TNSBatch(g, {0: t0, 1: t1}, {e: 2})
    with pytest.raises(RankMismatch):
        _compress_batch(st, e, 1e-12)


SQUARE = json.loads((GOLDEN / "square.json").read_text())["cases"]


@pytest.mark.parametrize("name", [c["name"] for c in SQUARE])
def test_cfg3_7x7_plan_bit_exact(name):
    """configs[3] family (7x7, reference default rank cap = treewidth bound + 1):
    path, score, cut plan, peak rank and multiplies equal the reference's."""
    case = next(c for c in SQUARE if c["name"] == name)
    r = case["results"][0]
    c, phi, psi, edges = _network(case, r["out"])
    n = c.num_qubits
    sn = _ShapeNet(range(n), edges)
    cuts = [tuple(e) for e in case["cuts"]] if case["cuts"] else None
    plan = _resolve_cuts(sn, cuts, case["max_rank"])
    path, score = _path_for(sn, plan, case["max_rank"])
    assert path == r["path"] and str(score) == r["path_score"]
    cp = ContractionPlan(NetworkSpec(list(range(n)), edges, {q: c.graph.node_edges(q) for q in range(n)}),
                         path, plan.cut_edges)
    assert cp.peak_rank == r["peak_rank"]
    assert str(cp.multiplies) == r["multiplies"]
    assert cp.slice_count == r["slice_count"]
