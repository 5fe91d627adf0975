"""Reference amplitudes of the 7x7 square-lattice circuit family (BASELINE
configs[3]: 49 qubits, gate set and pattern rule of configs[0]) at the depth the
reference can evaluate on CPU, written to tests/golden/square.json by running
the REFERENCE ``tnsim.compute_amplitude``
(/root/reference/pkg/src/tnsim/network.py:294-344) in this container:

    python tests/golden/make_golden_square.py

Cases (circuit = this repo's recipe builder, serialized and re-parsed by the
reference, seed 0 as in bench.py; max rank M = the reference's default,
treewidth bound + 1, network.py:320-321):

* 7x7, 8 cycles, two-sided (split 4), no cuts;
* the same with the explicit cut edges (20,27), (19,26) -- two of the cut edges
  of the depth-12 plan of bench.py's configs[3] entry (the slice loop,
  network.py:334-339).

A 49-qubit state vector does not exist; the reference's own contraction is
the oracle here.  /root/reference is not needed at test time.
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
    # name, rows, cols, depth, split, cuts, nbits
    ("cfg3_7x7_d8_twosided", 7, 7, 8, 4, None, 3),
    ("cfg3_7x7_d8_twosided_cut", 7, 7, 8, 4, [(20, 27), (19, 26)], 2),
]


def main():
    out_path = HERE / "square.json"
    doc = json.loads(out_path.read_text()) if out_path.exists() else {"cases": []}
    done = {c["name"] for c in doc["cases"]}
    rng = np.random.default_rng(49)
    for name, rows, cols, depth, split, cuts, nb in CASES:
        n = rows * cols
        outs = ["".join(rng.choice(["0", "1"], n)) for _ in range(nb)]
        if name in done:
            continue
        graph = mc.generate_lattice("square", rows, cols)
        circ = mc.pattern_rqc(graph, mc.square_patterns(rows, cols), depth, seed=0)
        text = mc.serialize_circuit(circ).decode()
        rcirc = rc.parse_circuit(text.encode())
        case = {"name": name, "rows": rows, "cols": cols, "depth": depth, "circuit": text, "in_bits": "0" * n,
                "split_cycle": split, "max_rank": None, "cuts": [list(e) for e in cuts] if cuts else None,
                "outs": outs, "results": []}
        for ob in outs:
            t0 = time.perf_counter()
            st = rn.compute_amplitude(rcirc, "0" * n, ob, split_cycle=split, cuts=cuts, max_rank=None)
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
