"""Generate the golden fixtures under tests/golden/ by running the REFERENCE
implementation (``tnsim`` from /root/reference/pkg/src) in this container.

    python tests/golden/make_golden.py

The fixtures pin both the CPU oracle (oracle/tn_oracle.py) and the GPU engine
to the reference's own outputs: amplitudes from ``compute_amplitude`` (default
two-sided split and the projected split == depth), state-vector amplitudes
from ``amplitude_oracle``, contraction paths/scores from ``find_optimal_path``,
cut plans from ``plan_cuts``, pairwise contractions from ``contract_pair``.
Circuits built with this repo's BASELINE-recipe builder are serialized and
re-parsed by the reference before use, so both sides see identical gates.
/root/reference is not needed at test time.
"""

from __future__ import annotations

import json
import random
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(HERE.parents[1]))

import tnsim  # noqa: E402  (reference)
from tnsim import circuit as rc  # noqa: E402
from tnsim import network as rn  # noqa: E402
from tnsim import pathfind as rp  # noqa: E402
from tnsim import tensor as rt  # noqa: E402
from tnsim.oracle import amplitude_oracle  # noqa: E402

import paper_2011_02621_b200.circuit as mc  # noqa: E402  (this repo's recipe builder)


def cplx(z):
    return [float(np.real(z)), float(np.imag(z))]


def edges_doc(edges: dict):
    return [[int(k), int(l), int(x)] for (k, l), x in sorted(edges.items())]


def bits_list(rng, n, count):
    return ["".join(rng.choice(["0", "1"], n)) for _ in range(count)]


def network_for(circ, in_bits, out_bits, split):
    fused = rc.fuse_single_qubit_gates(circ)
    phi, psi = tnsim.two_sided_evolve(fused, in_bits, out_bits, split)
    return rn.build_overlap_network(phi, psi)


def amplitude_case(name, circ, in_bits, outs, split, cuts, max_rank, with_sv=True):
    """Reference compute_amplitude for every bitstring (+ state vector)."""
    doc = {"name": name, "circuit": rc.serialize_circuit(circ).decode(), "in_bits": in_bits,
           "split_cycle": split, "cuts": cuts if not isinstance(cuts, list) else [list(e) for e in cuts],
           "max_rank": max_rank, "outs": outs, "results": []}
    net = network_for(circ, in_bits, outs[0], split)
    doc["edges"] = edges_doc(net.edges)
    for ob in outs:
        st = rn.compute_amplitude(circ, in_bits, ob, split_cycle=split,
                                  cuts=cuts if not isinstance(cuts, list) else [tuple(e) for e in cuts],
                                  max_rank=max_rank)
        rec = {"out": ob, "amplitude": cplx(st.amplitude), "path": st.path,
               "path_score": str(st.path_score), "peak_rank": st.peak_rank,
               "multiplies": str(st.multiplies), "slice_count": st.slice_count}
        if with_sv:
            rec["statevector"] = cplx(amplitude_oracle(circ, in_bits, ob))
        doc["results"].append(rec)
    return doc


def main():
    rng = np.random.default_rng(2011_02621)
    cases = []

    # BASELINE configs[0]: 3x3 square, 8 cycles, pattern sequence, no-repeat singles
    g = mc.generate_lattice("square", 3, 3)
    c0 = mc.pattern_rqc(g, mc.square_patterns(3, 3), 8, seed=0)
    circ0 = rc.parse_circuit(mc.serialize_circuit(c0))
    outs0 = bits_list(rng, 9, 64)
    cases.append(amplitude_case("cfg0_3x3_d8_projected", circ0, "0" * 9, outs0, 8, None, None))
    cases.append(amplitude_case("cfg0_3x3_d8_twosided", circ0, "0" * 9, outs0[:16], None, "auto", None))

    # reference generate_rqc circuits, several families / cut options
    for i, (kind, r, c, depth, fam, split, cuts, mr) in enumerate([
        ("square", 2, 3, 4, "fsim", None, "auto", None),
        ("square", 3, 3, 5, "fsim", None, "auto", 3),          # forces cuts (ref test)
        ("sycamore-like", 3, 3, 5, "fsim", None, None, None),
        ("sycamore-like", 3, 3, 5, "fsim", None, "explicit", None),
        ("square", 2, 4, 6, "iswap", 2, "auto", None),
        ("square", 3, 4, 6, "cz", None, "auto", 3),
        ("sycamore-like", 2, 5, 7, "fsim", 7, None, None),
        ("square", 3, 3, 6, "fsim", 6, [(1, 2), (4, 5)], None),
    ]):
        graph = rc.generate_lattice(kind, r, c)
        circ = rc.generate_rqc(graph, depth, seed=100 + i, gate_family=fam)
        n = graph.num_qubits
        if cuts == "explicit":
            cuts = [tuple(sorted(next(iter(sorted(graph.edges)))))]
        outs = bits_list(rng, n, 4)
        cases.append(amplitude_case(f"rqc{i}_{kind}_{r}x{c}_d{depth}_{fam}", circ, "0" * n, outs,
                                    split, cuts, mr))

    # configs[2]-style lattice (5x4) at a TNS-feasible depth, projected
    g = mc.generate_lattice("square", 5, 4)
    c2 = rc.parse_circuit(mc.serialize_circuit(mc.pattern_rqc(g, mc.square_patterns(5, 4), 6, seed=2)))
    cases.append(amplitude_case("cfg2_5x4_d6_projected", c2, "0" * 20, bits_list(rng, 20, 4), 6, None, None))

    (HERE / "amplitudes.json").write_text(json.dumps({"cases": cases}, indent=0))

    # ---------------- path search ----------------
    rnd = random.Random(7)
    paths = []

    def rand_shape(n):
        edges = set()
        for i in range(1, n):
            edges.add(rc.edge_key(rnd.randrange(i), i))
        for _ in range(rnd.randint(0, n)):
            a, b = rnd.sample(range(n), 2)
            edges.add(rc.edge_key(a, b))
        return rp.NetworkShape(tuple(range(n)), {e: rnd.choice([2, 4, 8]) for e in sorted(edges)})

    for t in range(60):
        shape = rand_shape(rnd.randint(3, 9))
        rec = {"edges": edges_doc(shape.edges), "n": len(shape.nodes), "runs": []}
        for opts in ({}, {"connectivity_pruning": False}, {"max_rank": 3}, {"max_rank": 4},
                     {"seeds": [0]}):
            try:
                p, s = rp.find_optimal_path(shape, **opts)
                rec["runs"].append({"opts": opts, "path": p, "score": str(s)})
            except rp.PathSearchError as e:
                rec["runs"].append({"opts": opts, "error": str(e), "largest": e.largest_subset})
        if len(shape.nodes) <= 8:
            p, s = rp.exhaustive_path_oracle(shape)
            rec["exhaustive"] = {"path": p, "score": str(s)}
        rec["treewidth"] = rp.treewidth_bound(shape)
        paths.append(rec)

    # lattice networks of the BASELINE recipes at scale (shape only)
    big = []
    for name, graph, pats, depth, splits, caps in [
        ("syc53_d12", *mc.sycamore53_graph()[:2], 12, (6, 12), (8,)),
        ("syc53_d8", *mc.sycamore53_graph()[:2], 8, (4, 8), (8,)),
        ("sq7x7_d8", mc.generate_lattice("square", 7, 7), mc.square_patterns(7, 7), 8, (4,), (9,)),
    ]:
        if isinstance(pats, dict):
            seq = "ABCDCDAB"
            pats = [pats[ch] for ch in seq]
        circ = mc.pattern_rqc(graph, pats, depth, seed=12)
        rcirc = rc.parse_circuit(mc.serialize_circuit(circ))
        for split in splits:
            fused = rc.fuse_single_qubit_gates(rcirc)
            n = rcirc.num_qubits
            phi, psi = tnsim.two_sided_evolve(fused, "0" * n, "0" * n, split)
            edges = {e: phi.bond_dims[e] * psi.bond_dims[e] for e in rcirc.graph.edges}
            shape = rp.NetworkShape(tuple(range(n)), edges)
            for cap in caps:
                p, s = rp.find_optimal_path(shape, cap)
                big.append({"name": name, "split": split, "cap": cap, "circuit_seed": 12,
                            "edges": edges_doc(edges), "path": p, "score": str(s),
                            "treewidth": rp.treewidth_bound(shape)})

    # plan_cuts on small overlap networks
    cutdocs = []
    for i, (kind, r, c, depth, cap) in enumerate([("square", 3, 4, 6, 3), ("square", 3, 3, 5, 3),
                                                   ("sycamore-like", 3, 4, 5, 4), ("square", 2, 3, 4, 10)]):
        graph = rc.generate_lattice(kind, r, c)
        circ = rc.generate_rqc(graph, depth, seed=6 if i == 0 else 20 + i)
        n = graph.num_qubits
        net = network_for(circ, "0" * n, "1" * n, None)
        try:
            plan = rn.plan_cuts(net, cap)
            cutdocs.append({"edges": edges_doc(net.edges), "cap": cap,
                            "cut_edges": [list(e) for e in plan.cut_edges], "slice_count": plan.slice_count})
        except rn.CutPlanError as e:
            cutdocs.append({"edges": edges_doc(net.edges), "cap": cap, "error": str(e)})
    (HERE / "paths.json").write_text(json.dumps({"random": paths, "lattice": big, "cuts": cutdocs}, indent=0))

    # ---------------- pairwise contractions + slicing ----------------
    arrays = {}
    meta = []
    for t in range(12):
        ra, rb = rnd.randint(1, 4), rnd.randint(1, 4)
        da = [rnd.randint(1, 4) for _ in range(ra)]
        db = [rnd.randint(1, 4) for _ in range(rb)]
        npairs = rnd.randint(0, min(ra, rb))
        pairs = list(zip(rnd.sample(range(ra), npairs), rnd.sample(range(rb), npairs)))
        for pa, pb in pairs:
            db[pb] = da[pa]
        a = rng.standard_normal(da) + 1j * rng.standard_normal(da)
        b = rng.standard_normal(db) + 1j * rng.standard_normal(db)
        out = rt.contract_pair(rt.Tensor(a, tuple(f"a{i}" for i in range(ra))),
                               rt.Tensor(b, tuple(f"b{i}" for i in range(rb))), pairs)
        arrays[f"a{t}"], arrays[f"b{t}"], arrays[f"out{t}"] = a, b, out.data
        meta.append({"pairs": [list(p) for p in pairs]})
    # slice_network golden on a small network
    graph = rc.generate_lattice("square", 2, 3)
    circ = rc.generate_rqc(graph, 4, seed=5)
    net = network_for(circ, "000000", "101010", None)
    plan = rn.plan_cuts(net, explicit_edges=[(1, 2), (3, 4)])
    for s in range(plan.slice_count):
        sl = rn.slice_network(net, plan, s)
        for q, tt in sl.tensors.items():
            arrays[f"slice{s}_node{q}"] = tt.data
    for q, tt in net.tensors.items():
        arrays[f"net_node{q}"] = tt.data
    meta_net = {"labels": {str(q): [list(e) for e in tt.labels] for q, tt in net.tensors.items()},
                "edges": edges_doc(net.edges), "cut_edges": [[1, 2], [3, 4]], "slice_count": plan.slice_count,
                "whole": cplx(rn.contract_along_path(net, sorted(net.tensors))[0])}
    np.savez_compressed(HERE / "pairs.npz", **arrays)
    (HERE / "pairs.json").write_text(json.dumps({"pairs": meta, "net": meta_net}, indent=0))
    print("wrote", [p.name for p in HERE.iterdir()])


if __name__ == "__main__":
    main()
