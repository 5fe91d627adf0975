"""The cut plans bench.py reports are what its config strings say (host only):
slice counts, largest intermediates and multiply counts of the headline plan,
the nested 2^31 and depth-11 plans and the configs[2]/[3] entries, with the
path re-searched on the slice-0 estimate as the reference does
(network.py:323-330)."""

import sys

import pytest

from conftest import ROOT

sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tools"))

import bench  # noqa: E402
from cut_search import network_shape  # noqa: E402
from paper_2011_02621_b200.engine import ContractionPlan, NetworkSpec  # noqa: E402
from paper_2011_02621_b200.pathfind import NetworkShape, find_optimal_path  # noqa: E402


def _plan(net, depth, split, cuts, cap, rows=0, cols=0):
    edges, legs = network_shape(net, depth, split, rows, cols, seed=bench.SEED)
    est = dict(edges)
    for e in cuts:
        est[e] = 1
    n = len(legs)
    path, _ = find_optimal_path(NetworkShape(tuple(range(n)), est), cap)
    return ContractionPlan(NetworkSpec(list(range(n)), edges, legs), path, cuts)


@pytest.mark.parametrize("pc,mult", [(bench.D12, 15042767638496256), (bench.D12_CAP31, 19937040619601920),
                                     (bench.D11, 445092594713088)])
def test_sycamore_plans(pc, mult):
    plan = _plan("syc53", pc["depth"], pc["split"], pc["cuts"], pc["cap"])
    assert plan.slice_count == pc["slices"]
    assert plan.max_elems == 1 << pc["elem_log2"]
    assert plan.multiplies == mult


@pytest.mark.parametrize("name,slices,elems,mult", [
    ("amplitudes_cfg2_d14", 1, 1 << 31, None),
    ("amplitudes_cfg2_d16", 16384, 1 << 29, 226609415472545792),
    ("amplitudes_cfg3_d10", 1, 1 << 33, None),
    ("amplitudes_cfg3_d12", 1 << 20, 1 << 30, 2097555926641803264),
])
def test_square_plans(name, slices, elems, mult):
    c = bench.SQUARE[name]
    plan = _plan("square", c["depth"], c["split"], c["cuts"] or [], c["cap"], c["rows"], c["cols"])
    assert plan.slice_count == slices
    assert plan.max_elems == elems
    if mult is not None:
        assert plan.multiplies == mult
