"""Numpy interpreter of the engine's device descriptors (test infrastructure).

Executes a ``ContractionPlan`` exactly as libtnc's kernels are specified in
include/tnc.h -- site re-layout, projection gather with slice offsets, every
step through its row map / offset tables, slice sum -- so the host planner's
layouts can be validated on a CPU-only box against the oracle.
"""

from __future__ import annotations

from math import prod

import numpy as np

from paper_2011_02621_b200.engine import _mixed, _site_cut_info, _strides


def _row_offsets(fd, fa, fc, M):
    f = np.arange(M, dtype=np.int64)
    oa = np.zeros(M, dtype=np.int64)
    oc = np.zeros(M, dtype=np.int64)
    for d, a, c in zip(reversed(fd), reversed(fa), reversed(fc)):
        r = f % d
        f //= d
        oa += r * a
        oc += r * c
    return oa, oc


def _slice_off(cuts, s):
    return sum(((s // div) % ext) * st for st, div, ext in cuts)


def run_plan(plan, sites: dict, sel: dict | None, B: int, slices=None) -> np.ndarray:
    spec = plan.spec
    slices = range(plan.slice_count) if slices is None else slices
    amps = np.zeros(B, dtype=np.complex128)
    # per-step re-laid-out sites
    prepared = []
    for sp in plan.steps:
        q = sp.node
        sdims = spec.site_dims(q)
        sstr = dict(zip(spec.legs[q], _strides(sdims)))
        ldims = [int(spec.edges[e]) for e in sp.site_layout]
        offs = _mixed(ldims, [sstr[e] for e in sp.site_layout])
        raw = sites[q].reshape(sites[q].shape[0], -1)
        prepared.append((raw[:, offs], _site_cut_info(plan, sp.site_layout, ldims)))
    q0 = plan.path[0]
    sdims0 = spec.site_dims(q0)
    sstr0 = dict(zip(spec.legs[q0], _strides(sdims0)))
    first_off = _mixed(plan.first_dims, [sstr0[e] for e in plan.first_legs])
    cuts0 = _site_cut_info(plan, spec.legs[q0], sdims0)
    raw0 = sites[q0].reshape(sites[q0].shape[0], -1)
    for b in range(B):
        for s in slices:
            v0 = int(sel[q0][b]) if sel is not None and raw0.shape[0] > 1 else 0
            acc = raw0[v0][_slice_off(cuts0, s) + first_off]
            for sp, (site, cuts) in zip(plan.steps, prepared):
                v = int(sel[sp.node][b]) if sel is not None and site.shape[0] > 1 else 0
                S = site[v][_slice_off(cuts, s) + np.arange(sp.K * sp.N)].reshape(sp.K, sp.N)
                A = acc.reshape(sp.M, sp.K)            # a_rows_contig by construction
                res = A @ S
                oa, oc = _row_offsets(sp.f_dim, sp.f_astride, sp.f_cstride, sp.M)
                out = np.zeros(sp.M * sp.N, dtype=np.complex128)
                out[(oc[:, None] + sp.c_noff[None, :]).reshape(-1)] = res.reshape(-1)
                # the row map must agree with plain row order on the acc side
                assert np.array_equal(oa, np.arange(sp.M) * sp.K)
                acc = out
            amps[b] += acc.reshape(-1)[0]
    return amps
