"""Reference amplitudes of the 53-qubit Sycamore circuit family (BASELINE
configs[4]: 53-qubit diagonal lattice, ABCDCDAB, fSim(pi/2, pi/6)) at the
depths the reference itself can evaluate on CPU, written to
tests/golden/syc53.json by running the REFERENCE ``tnsim.compute_amplitude``
(/root/reference/pkg/src/tnsim/network.py:294-344) in this container:

    python tests/golden/make_golden_syc53.py [--quick]

Cases (circuit = this repo's recipe builder, serialized and re-parsed by the
reference, seed 0 as in bench.py):

* projected (split_cycle = depth), depths 6 and 7, rank cap 12, no cuts;
* projected depth 8 with the cut edges of bench.py's sliced plan (64 slices);
* two-sided (split = depth // 2), depth 8, rank cap 12, no cuts;
* two-sided depth 8 with the cut edges of the depth-12 plan (45,49), (38,45) --
  the same two-sided slicing scheme the depth-12 measurement uses.

Each record keeps the reference's amplitude, path, path score, peak rank,
multiply count and slice count.  /root/reference is not needed at test time.
"""

from __future__ import annotations

import json
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(HERE.parents[1]))

from tnsim import circuit as rc  # noqa: E402  (reference)
from tnsim import network as rn  # noqa: E402

import paper_2011_02621_b200.circuit as mc  # noqa: E402  (this repo's recipe builder)

CASES = [
    # name, depth, split, cuts, nbits
    ("syc53_d6_projected", 6, 6, None, 4),
    ("syc53_d7_projected", 7, 7, None, 2),
    ("syc53_d8_twosided", 8, 4, None, 4),
    ("syc53_d8_twosided_cut", 8, 4, [(45, 49), (38, 45)], 2),
    ("syc53_d8_projected_cut", 8, 8, [(9, 14), (2, 9)], 1),
]


def main():
    quick = "--quick" in sys.argv
    out_path = HERE / "syc53.json"
    doc = json.loads(out_path.read_text()) if out_path.exists() else {"cases": []}
    done = {c["name"] for c in doc["cases"]}
    rng = np.random.default_rng(53)
    graph, pats, _ = mc.sycamore53_graph()
    for name, depth, split, cuts, nb in CASES:
        outs = ["".join(rng.choice(["0", "1"], 53)) for _ in range(nb)]
        if name in done or (quick and depth >= 8 and split == depth):
            continue
        circ = mc.pattern_rqc(graph, [pats[c] for c in "ABCDCDAB"], depth, seed=0)
        text = mc.serialize_circuit(circ).decode()
        rcirc = rc.parse_circuit(text.encode())
        case = {"name": name, "circuit": text, "in_bits": "0" * 53, "split_cycle": split, "max_rank": 12,
                "cuts": [list(e) for e in cuts] if cuts else None, "outs": outs, "results": []}
        for ob in outs:
            t0 = time.perf_counter()
            st = rn.compute_amplitude(rcirc, "0" * 53, ob, split_cycle=split, cuts=cuts, max_rank=12)
            rec = {"out": ob, "amplitude": [float(st.amplitude.real), float(st.amplitude.imag)],
                   "path": st.path, "path_score": str(st.path_score), "peak_rank": st.peak_rank,
                   "multiplies": str(st.multiplies), "slice_count": st.slice_count,
                   "reference_wall_s": time.perf_counter() - t0}
            case["results"].append(rec)
            print(name, ob[:12], rec["amplitude"], f"{rec['reference_wall_s']:.1f}s", flush=True)
        doc["cases"].append(case)
        out_path.write_text(json.dumps(doc, indent=0))


if __name__ == "__main__":
    main()
