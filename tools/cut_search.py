"""Greedy cut-edge search for sliced amplitude networks (host only).

The reference's ``plan_cuts`` (network.py:173-215) bounds the path's *rank*
and, on the 53-qubit networks, fails (it cuts every Fiedler separator and the
path search still exceeds the cap).  The BASELINE configs cap intermediates
at 2^30 *elements*, so this tool picks the cut set; everything after it follows
the reference exactly: the path is ``find_optimal_path`` on the slice-0
estimate (cut edges at extent 1, network.py:323-330) and every slice is
contracted along it.

Greedy rule: each round tries every uncut edge, re-runs the path search on
the sliced estimate, and keeps the edge with the least increase of
log2(total multiplies) per halving of the largest intermediate; a final pass
drops any cut that is no longer needed.

    python tools/cut_search.py --net syc53 --depth 12 --split 6 --target 30 [--cap 12] [--json out]
    python tools/cut_search.py --net square --rows 5 --cols 4 --depth 16 --split 8 --target 30
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import time
from multiprocessing import Pool

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2011_02621_b200.circuit import (fuse_single_qubit_gates, generate_lattice,  # noqa: E402
                                           pattern_rqc, square_patterns, sycamore53_graph)
from paper_2011_02621_b200.engine import ContractionPlan, NetworkSpec  # noqa: E402
from paper_2011_02621_b200.pathfind import NetworkShape, PathSearchError, find_optimal_path  # noqa: E402
from paper_2011_02621_b200.tns import two_sided_evolve  # noqa: E402

_G = {}


def network_shape(net: str, depth: int, split: int, rows=0, cols=0, seed=0):
    """(edges, legs) of the overlap network <0..0|U|0..0> (two-sided at ``split``;
    split == depth is the projected network).  Bond dims do not depend on the
    bitstring for these circuits (checked by tests/test_twosided.py)."""
    if net == "syc53":
        graph, pats, _ = sycamore53_graph()
        circ = pattern_rqc(graph, [pats[c] for c in "ABCDCDAB"], depth, seed=seed)
    else:
        graph = generate_lattice("square", rows, cols)
        circ = pattern_rqc(graph, square_patterns(rows, cols), depth, seed=seed)
    fused = fuse_single_qubit_gates(circ)
    n = fused.graph.num_qubits
    phi, psi = two_sided_evolve(fused, "0" * n, "0" * n, split)
    edges = {e: phi.bond_dims[e] * psi.bond_dims[e] for e in fused.graph.edges}
    legs = {q: fused.graph.node_edges(q) for q in range(n)}
    return edges, legs


def evaluate(cuts):
    edges, legs, cap = _G["edges"], _G["legs"], _G["cap"]
    est = dict(edges)
    for e in cuts:
        est[e] = 1
    n = len(legs)
    try:
        path, score = find_optimal_path(NetworkShape(tuple(range(n)), est), cap)
    except PathSearchError:
        return None
    plan = ContractionPlan(NetworkSpec(list(range(n)), edges, legs), path, cuts)
    return {"cuts": [list(e) for e in cuts], "max_elems": plan.max_elems, "multiplies": plan.multiplies,
            "slices": plan.slice_count, "path": path, "score": score}


def beam_search(pool, edges, root, args):
    def key(r):
        return math.log2(r["multiplies"]) + max(0.0, math.log2(r["max_elems"]) - args.target)

    beams, best, seen = [root], None, set()
    for level in range(args.max_cuts):
        jobs = []
        for b in beams:
            have = [tuple(e) for e in b["cuts"]]
            for e in sorted(edges):
                if e in have or edges[e] <= 1:
                    continue
                fs = frozenset(have + [e])
                if fs in seen:
                    continue
                seen.add(fs)
                jobs.append(have + [e])
        res = [r for r in pool.map(evaluate, jobs) if r is not None]
        for r in res:
            if math.log2(r["max_elems"]) <= args.target + 1e-9 and (best is None or r["multiplies"] < best["multiplies"]):
                best = r
        res.sort(key=key)
        beams = [r for r in res if best is None or r["multiplies"] < best["multiplies"]][: args.beam]
        print(f"level {level + 1}: {len(jobs)} sets; best beam " +
              ", ".join(f"{[tuple(e) for e in r['cuts']]} 2^{math.log2(r['max_elems']):.1f} {r['multiplies']:.3e}"
                        for r in beams[:3]) +
              (f"; best solution {best['cuts']} {best['multiplies']:.3e}" if best else ""), flush=True)
        if not beams:
            break
    if best is None:
        raise SystemExit("beam search found no cut set under the target")
    return best


def _init(edges, legs, cap):
    _G.update(edges=edges, legs=legs, cap=cap)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--net", default="syc53", choices=["syc53", "square"])
    ap.add_argument("--rows", type=int, default=5)
    ap.add_argument("--cols", type=int, default=4)
    ap.add_argument("--depth", type=int, default=12)
    ap.add_argument("--split", type=int, default=6)
    ap.add_argument("--cap", type=int, default=12)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--target", type=float, default=30.0, help="log2 of the largest intermediate")
    ap.add_argument("--procs", type=int, default=os.cpu_count())
    ap.add_argument("--json", default=None)
    ap.add_argument("--beam", type=int, default=0,
                    help="beam search of this width (0: greedy); beams ranked by "
                         "log2(multiplies) + max(0, log2(largest) - target)")
    ap.add_argument("--max-cuts", type=int, default=6)
    ap.add_argument("--init-cuts", default="", help="start from these cut edges, e.g. 45-49,38-45")
    args = ap.parse_args()
    edges, legs = network_shape(args.net, args.depth, args.split, args.rows, args.cols, args.seed)
    _init(edges, legs, args.cap)
    t0 = time.time()
    cur = evaluate([])
    print(f"unsliced: 2^{math.log2(cur['max_elems']):.1f} elems, {cur['multiplies']:.3e} mult", flush=True)
    cuts = [tuple(int(x) for x in c.split("-")) for c in args.init_cuts.split(",")] if args.init_cuts else []
    if cuts:
        cur = evaluate(cuts)
        print(f"initial {cuts}: 2^{math.log2(cur['max_elems']):.1f} elems, {cur['multiplies']:.3e} mult", flush=True)
    if args.beam:
        with Pool(args.procs, initializer=_init, initargs=(edges, legs, args.cap)) as pool:
            cur = beam_search(pool, edges, cur, args)
        cuts = [tuple(e) for e in cur["cuts"]]
    with Pool(args.procs, initializer=_init, initargs=(edges, legs, args.cap)) as pool:
        while math.log2(cur["max_elems"]) > args.target + 1e-9:
            cand = [e for e in sorted(edges) if e not in cuts and edges[e] > 1]
            res = pool.map(evaluate, [cuts + [e] for e in cand])
            best, best_key = None, None
            for e, r in zip(cand, res):
                if r is None or r["max_elems"] >= cur["max_elems"]:
                    continue
                gain = math.log2(cur["max_elems"]) - math.log2(r["max_elems"])
                cost = math.log2(r["multiplies"]) - math.log2(cur["multiplies"])
                key = (max(cost, 0.0) / gain, -gain, e)
                if best_key is None or key < best_key:
                    best, best_key = (e, r), key
            if best is None:
                raise SystemExit("no cut reduces the largest intermediate")
            cuts.append(best[0])
            cur = best[1]
            print(f"+{best[0]} (dim {edges[best[0]]}): 2^{math.log2(cur['max_elems']):.1f} elems, "
                  f"{cur['multiplies']:.3e} mult, {cur['slices']} slices  [{time.time() - t0:.0f}s]", flush=True)
        # prune cuts that became redundant
        changed = True
        while changed:
            changed = False
            trial = [[c for c in cuts if c != e] for e in cuts]
            res = pool.map(evaluate, trial)
            for t, r in sorted(zip(trial, res), key=lambda x: (x[1] or {"multiplies": 1e99})["multiplies"]):
                if r is not None and math.log2(r["max_elems"]) <= args.target + 1e-9 and \
                        r["multiplies"] <= cur["multiplies"]:
                    cuts, cur, changed = t, r, True
                    print(f"pruned -> {len(cuts)} cuts, {cur['multiplies']:.3e} mult", flush=True)
                    break
    cur["net"] = vars(args)
    cur["score"] = str(cur["score"])
    print(json.dumps({k: v for k, v in cur.items() if k != "path"}), flush=True)
    if args.json:
        with open(args.json, "w") as f:
            json.dump(cur, f, indent=1)


if __name__ == "__main__":
    main()
