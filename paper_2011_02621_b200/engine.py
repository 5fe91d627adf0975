"""Batched contraction engine: host planner + device executor.

The engine evaluates ``contract_along_path`` (reference network.py:246-268)
for a batch of output bitstrings and all slices of a cut plan at once.  Every
batch element z = (bitstring b, slice s) contracts the same network shape along
the same path; only the *projected site tensors* differ:

    site(q, z) = T_q[sel[q, b]] with cut legs fixed to their slice values,

where ``T_q`` has a leading variant axis (2 variants = the projected physical
index in projected mode, one per bitstring in two-sided mode, 1 for a plain
network).

Planning (host, once per network/path/cut plan):

* accumulator legs are kept ordered by *due step* -- the path position of the
  node on their far side, latest outermost -- so the legs contracted at every
  step are the innermost, contiguous ones: the accumulator is always a plain
  row-major [M, K] matrix per batch element (no permute pass ever);
* each step's site tensor is re-laid out once on the device as
  [variant, cut legs, shared legs (acc order), new legs (out order)], i.e. a
  dense [K][N] block per (variant, slice);
* the result legs are again due-ordered; when all new legs fall innermost the
  result is a plain [M, N] matrix (``c_rows_contig``), otherwise the kernels
  scatter rows through a mixed-radix row map plus an N table.

Execution (device): one ``tnc_contract_path`` call per (bitstring x slice)
chunk -- projection gather, every step, deterministic slice sum.  There is no
host fallback: without ``libtnc.so`` or an sm_100 device the engine raises.
"""

from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from math import prod
from typing import Sequence

import numpy as np

from . import _native as NV

Edge = tuple

__all__ = ["NetworkSpec", "ContractionPlan", "PathExecutor", "EngineError",
           "device_contract_pair", "contract_pair_device", "dtype_code"]


class EngineError(RuntimeError):
    pass


def dtype_code(dtype: str) -> int:
    if dtype in ("complex64", "c64"):
        return NV.C64
    if dtype in ("complex128", "c128"):
        return NV.C128
    raise EngineError(f"unsupported dtype {dtype!r} (complex64 | complex128)")


@dataclass
class NetworkSpec:
    """Closed network shape: nodes, edge extents, leg order of each site tensor."""

    nodes: list
    edges: dict
    legs: dict

    def __post_init__(self):
        seen: dict = {}
        for q in self.nodes:
            for e in self.legs[q]:
                if e not in self.edges:
                    raise EngineError(f"node {q}: leg {e} is not a network edge")
                if q not in e:
                    raise EngineError(f"node {q}: leg {e} does not touch it")
                seen[e] = seen.get(e, 0) + 1
        if any(c != 2 for c in seen.values()) or set(seen) != set(self.edges):
            raise EngineError("network is not closed")

    def site_dims(self, q) -> tuple:
        return tuple(int(self.edges[e]) for e in self.legs[q])


def _strides(dims: Sequence[int]) -> list[int]:
    out, s = [0] * len(dims), 1
    for i in range(len(dims) - 1, -1, -1):
        out[i] = s
        s *= int(dims[i])
    return out


def _mixed(dims: Sequence[int], strides: Sequence[int]) -> np.ndarray:
    """Offsets of every mixed-radix index over ``dims`` (outermost first)."""
    off = np.zeros(1, dtype=np.int64)
    for d, s in zip(dims, strides):
        off = (off[:, None] + np.arange(int(d), dtype=np.int64)[None, :] * int(s)).reshape(-1)
    return off


def _merge_rows(dims, astr, cstr):
    """Fuse adjacent free legs that are contiguous in both acc and out."""
    md, ma, mc = [], [], []
    for d, a, c in zip(dims, astr, cstr):
        if d == 1:
            continue
        if md and ma[-1] == a * d and mc[-1] == c * d:
            md[-1] *= d
            ma[-1] = a
            mc[-1] = c
        else:
            md.append(d)
            ma.append(a)
            mc.append(c)
    return md, ma, mc


@dataclass
class StepPlan:
    node: int
    acc_legs: list            # legs of the accumulator before the step
    shared: list
    free: list
    new: list
    out_legs: list
    M: int
    K: int
    N: int
    c_rows_contig: bool
    f_dim: list = field(default_factory=list)
    f_astride: list = field(default_factory=list)
    f_cstride: list = field(default_factory=list)
    c_noff: np.ndarray = None
    site_layout: list = None  # [cut legs..., shared..., new...]
    n_dim: list = field(default_factory=list)      # new legs (site order, merged), result strides
    n_cstride: list = field(default_factory=list)


class ContractionPlan:
    """Static plan for one network shape, path and cut plan."""

    def __init__(self, spec: NetworkSpec, path: Sequence[int], cut_edges: Sequence[Edge] = ()):
        if sorted(path) != sorted(spec.nodes):
            raise ValueError("path is not a permutation of the network's qubits")
        self.spec = spec
        self.path = list(path)
        self.cut = [tuple(e) for e in cut_edges]
        if len(set(self.cut)) != len(self.cut):
            raise ValueError("duplicate cut edges")
        for e in self.cut:
            if e not in spec.edges:
                raise ValueError(f"cut edge {e} not in network")
        self.cut_ext = [int(spec.edges[e]) for e in self.cut]
        self.slice_count = prod(self.cut_ext) if self.cut else 1
        # mixed radix, first cut edge most significant (network.py:228-232)
        self.cut_div = {}
        div = 1
        for e, x in zip(reversed(self.cut), reversed(self.cut_ext)):
            self.cut_div[e] = div
            div *= x
        cutset = set(self.cut)
        pos = {q: i for i, q in enumerate(self.path)}
        self.pos = pos

        def other(e, q):
            return e[1] if e[0] == q else e[0]

        def due_key(e, q):
            return (-pos[other(e, q)], e)

        ext = {e: int(x) for e, x in spec.edges.items()}
        q0 = self.path[0]
        acc = sorted((e for e in spec.legs[q0] if e not in cutset), key=lambda e: due_key(e, q0))
        # owner[e] = included endpoint of an open accumulator leg
        owner = {e: q0 for e in acc}
        self.first_legs = list(acc)
        self.first_dims = [ext[e] for e in acc]
        self.steps: list[StepPlan] = []
        peak = sum(1 for e in acc if ext[e] > 1)
        max_elems = prod(self.first_dims) if acc else 1
        mult = 0
        for t in range(1, len(self.path)):
            q = self.path[t]
            shared = [e for e in acc if other(e, owner[e]) == q]
            ns = len(shared)
            if acc[len(acc) - ns:] != shared:
                raise EngineError("internal: shared legs are not innermost")
            free = acc[: len(acc) - ns]
            new = [e for e in spec.legs[q] if e not in cutset and e not in shared]
            for e in new:
                owner[e] = q
            out = sorted(free + new, key=lambda e: due_key(e, owner[e]))
            new_out = [e for e in out if e in set(new)]
            M = prod(ext[e] for e in free) if free else 1
            K = prod(ext[e] for e in shared) if shared else 1
            N = prod(ext[e] for e in new_out) if new_out else 1
            adims = [ext[e] for e in acc]
            astr = dict(zip(acc, _strides(adims)))
            odims = [ext[e] for e in out]
            ostr = dict(zip(out, _strides(odims)))
            c_contig = out == free + new_out
            fd, fa, fc = _merge_rows([ext[e] for e in free], [astr[e] for e in free], [ostr[e] for e in free])
            nd_, _, nc_ = _merge_rows([ext[e] for e in new_out], [ostr[e] for e in new_out], [ostr[e] for e in new_out])
            sp = StepPlan(
                node=q, acc_legs=list(acc), shared=shared, free=free, new=new_out, out_legs=out,
                M=M, K=K, N=N, c_rows_contig=c_contig, f_dim=fd, f_astride=fa, f_cstride=fc,
                c_noff=_mixed([ext[e] for e in new_out], [ostr[e] for e in new_out]),
                site_layout=[e for e in self.cut if e in set(spec.legs[q])] + shared + new_out,
                n_dim=nd_, n_cstride=nc_,
            )
            if len(fd) > NV.MAX_LEGS:
                raise EngineError(f"step {t}: {len(fd)} free legs exceed TNC_MAX_LEGS")
            self.steps.append(sp)
            mult += M * K * N
            acc = out
            for e in shared:
                owner.pop(e, None)
            peak = max(peak, sum(1 for e in acc if ext[e] > 1))
            max_elems = max(max_elems, prod(odims) if out else 1)
        if acc:
            raise EngineError("internal: accumulator not closed at the end of the path")
        self.peak_rank = peak
        self.max_elems = max_elems
        self.multiplies_per_slice = mult
        self.multiplies = mult * self.slice_count

    # -- roofline bookkeeping -------------------------------------------------
    def step_traffic(self, itemsize: int):
        """(algorithmic bytes, flops) per batch element for every step."""
        out = []
        for sp in self.steps:
            bytes_ = (sp.M * sp.K + sp.M * sp.N) * itemsize
            out.append((bytes_, 8 * sp.M * sp.K * sp.N))
        return out


def _site_cut_info(plan: ContractionPlan, layout: Sequence[Edge], dims: Sequence[int]):
    """(cut_stride, cut_div, cut_ext) for the cut legs present in ``layout``."""
    st = dict(zip(layout, _strides(dims)))
    info = []
    for e in plan.cut:
        if e in st:
            info.append((st[e], plan.cut_div[e], int(plan.spec.edges[e])))
    return info


def _fill_site(site: NV.Site, ptr: int, vstride: int, cuts, nvariants: int = 0) -> None:
    site.ptr = ptr
    site.sel = None
    site.zstride = 0
    site.vstride = vstride
    site.nvariants = nvariants
    site.ncut = len(cuts)
    if len(cuts) > NV.MAX_CUTS:
        raise EngineError(f"{len(cuts)} cut legs on one site exceed TNC_MAX_CUTS")
    for i, (s, d, x) in enumerate(cuts):
        site.cut_stride[i] = s
        site.cut_div[i] = d
        site.cut_ext[i] = x


class PathExecutor:
    """Device state for one plan: re-laid-out site tensors, offset tables,
    ping-pong accumulators; ``run`` evaluates amplitudes for a bitstring batch."""

    def __init__(self, plan: ContractionPlan, sites: dict, dtype: str = "complex128",
                 device=None, max_batch_elems: int | None = None):
        import torch

        NV.require_device()
        self.torch = torch
        self.plan = plan
        self.dtype = dtype
        self.code = dtype_code(dtype)
        self.tdtype = torch.complex64 if self.code == NV.C64 else torch.complex128
        self.itemsize = 8 if self.code == NV.C64 else 16
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        spec = plan.spec
        L = NV.lib()
        stream = torch.cuda.current_stream(self.device).cuda_stream
        self.raw = {}
        self.nvar = {}
        self.step_sites = []
        self.load_sites(sites, stream)
        # offset tables
        self.tables = []
        for sp in plan.steps:
            K, N = sp.K, sp.N
            tab = np.concatenate([
                np.arange(K, dtype=np.int64),
                np.arange(K, dtype=np.int64) * N,
                np.arange(N, dtype=np.int64),
                sp.c_noff.astype(np.int64),
            ])
            self.tables.append(torch.from_numpy(tab).to(self.device))
        torch.cuda.synchronize(self.device)
        # batch sizing: two accumulators of max_elems per batch element
        if max_batch_elems is None:
            free, _ = torch.cuda.mem_get_info(self.device)
            max_batch_elems = max(1, int(0.35 * free) // (2 * self.itemsize * plan.max_elems))
        self.max_z = max(1, int(max_batch_elems))
        self._buf = None
        self._graphs: dict = {}
        self._graph_seen: set = set()
        self._build_descs()

    def load_sites(self, sites: dict, stream=None) -> None:
        """(Re)load the raw site tensors [V, dims...] and re-lay them out per
        step ([V, cut legs, shared legs, new legs]) with the projection kernel.
        A reload with the same variant counts writes into the existing step
        blocks, so descriptors (and captured graphs) stay valid."""
        torch = self.torch
        plan, spec = self.plan, self.plan.spec
        L = NV.lib()
        st = torch.cuda.current_stream(self.device) if stream is None else stream
        sptr = st if isinstance(st, int) else st.cuda_stream
        reload = bool(self.step_sites)
        for q in spec.nodes:
            t = sites[q]
            if not isinstance(t, torch.Tensor):
                t = torch.from_numpy(np.ascontiguousarray(t))
            t = t.to(device=self.device, dtype=self.tdtype).contiguous()
            dims = spec.site_dims(q)
            if tuple(t.shape[1:]) != dims:
                raise EngineError(f"site {q}: shape {tuple(t.shape)} != (V, {dims})")
            if reload:
                if int(t.shape[0]) != self.nvar[q]:
                    raise EngineError(f"site {q}: {int(t.shape[0])} variants, executor holds {self.nvar[q]}")
                self.raw[q].copy_(t)             # in place: pointers in descriptors / graphs stay valid
                continue
            self.raw[q] = t
            self.nvar[q] = int(t.shape[0])
        for i, sp in enumerate(plan.steps):
            q = sp.node
            legs = spec.legs[q]
            sdims = spec.site_dims(q)
            sstr = dict(zip(legs, _strides(sdims)))
            ldims = [int(spec.edges[e]) for e in sp.site_layout]
            V = self.nvar[q]
            per_var = prod(sdims) if sdims else 1
            new_per_var = prod(ldims) if ldims else 1
            if reload:
                dst = self.step_sites[i][0]
            else:
                dst = torch.empty((V, new_per_var), dtype=self.tdtype, device=self.device)
            d = NV.ProjectDesc()
            d.dtype = self.code
            d.conj = 0
            d.Z = V
            d.slices_per_b = 1
            d.s0 = 0
            _fill_site(d.site, self.raw[q].data_ptr(), 0, [])
            d.site.zstride = per_var
            d.out = dst.data_ptr()
            d.out_zstride = new_per_var
            d.nd = len(ldims)
            for j, e in enumerate(sp.site_layout):
                d.dim[j] = ldims[j]
                d.src_stride[j] = sstr[e]
            NV.check(L.tnc_project(C.byref(d), C.c_void_p(sptr)), "site relayout")
            if not reload:
                self.step_sites.append((dst, new_per_var, _site_cut_info(plan, sp.site_layout, ldims)))

    def _build_descs(self):
        plan, spec = self.plan, self.plan.spec
        q0 = plan.path[0]
        legs = spec.legs[q0]
        sdims = spec.site_dims(q0)
        sstr = dict(zip(legs, _strides(sdims)))
        pd = NV.PathDesc()
        f = pd.first
        f.dtype = self.code
        f.conj = 0
        per_var = prod(sdims) if sdims else 1
        _fill_site(f.site, self.raw[q0].data_ptr(), per_var,
                   _site_cut_info(plan, legs, sdims))
        f.nd = len(plan.first_legs)
        for i, e in enumerate(plan.first_legs):
            f.dim[i] = int(spec.edges[e])
            f.src_stride[i] = sstr[e]
        steps = (NV.StepDesc * max(1, len(plan.steps)))()
        for i, sp in enumerate(plan.steps):
            d = steps[i]
            d.dtype = self.code
            d.kernel = NV.K_AUTO
            dst, per_var, cuts = self.step_sites[i]
            _fill_site(d.site, dst.data_ptr(), per_var, cuts, self.nvar[sp.node])
            d.M, d.K, d.N = sp.M, sp.K, sp.N
            d.nf = len(sp.f_dim)
            for j in range(d.nf):
                d.f_dim[j] = sp.f_dim[j]
                d.f_astride[j] = sp.f_astride[j]
                d.f_cstride[j] = sp.f_cstride[j]
            tab = self.tables[i]
            base = tab.data_ptr()
            d.a_koff = base
            d.b_koff = base + 8 * sp.K
            d.b_noff = base + 16 * sp.K
            d.c_noff = base + 16 * sp.K + 8 * sp.N
            d.a_rows_contig = 1
            d.c_rows_contig = 1 if sp.c_rows_contig else 0
            d.c_n_contig = 1 if np.array_equal(sp.c_noff, np.arange(sp.N)) else 0
            d.nn = len(sp.n_dim) if len(sp.n_dim) <= NV.MAX_LEGS else 0
            for j in range(d.nn):
                d.n_dim[j] = sp.n_dim[j]
                d.n_cstride[j] = sp.n_cstride[j]
            d.b_dense = 1
            d.conj_b = 0
        # complex64 tensor-core GEMM steps take their input's per-z magnitude
        # bound from the previous step (amax_out -> amax_in, two ping-pong
        # rows), which lets them run fp16-split MMAs (tnc.h, tnc_tcgemm.cuh)
        self._amax = None
        if self.code == NV.C64 and len(plan.steps) > 1:
            self._amax = self.torch.zeros((2, self.max_z), dtype=self.torch.float32, device=self.device)
            for i in range(1, len(plan.steps)):
                sp = plan.steps[i]
                if sp.K % 16 == 0 and sp.K * sp.N >= 256:
                    ptr = self._amax[i & 1].data_ptr()
                    steps[i].amax_in = ptr
                    steps[i - 1].amax_out = ptr
        pd.nsteps = len(plan.steps)
        pd.steps = C.cast(steps, C.POINTER(NV.StepDesc))
        pd.reduce.dtype = self.code
        self._pd = pd
        self._steps = steps

    def _buffers(self, z: int):
        torch = self.torch
        need = z * self.plan.max_elems
        if self._buf is None or self._buf[0].numel() < need:
            # captured graphs hold the old accumulator pointers: drop them with
            # the buffers they write (a replay would otherwise write freed memory)
            self._graphs.clear()
            self._graph_seen.clear()
            self._buf = None
            self._buf = (torch.empty(need, dtype=self.tdtype, device=self.device),
                         torch.empty(need, dtype=self.tdtype, device=self.device))
        return self._buf

    def chunks(self, B: int, slices: range):
        """(b0, nb, s0, ns) work chunks covering B bitstrings x ``slices``."""
        S = len(slices)
        out = []
        if S <= self.max_z:
            nb = max(1, self.max_z // S)
            for b0 in range(0, B, nb):
                out.append((b0, min(nb, B - b0), slices.start, S))
        else:
            for b0 in range(B):
                for s0 in range(slices.start, slices.stop, self.max_z):
                    out.append((b0, 1, s0, min(self.max_z, slices.stop - s0)))
        return out

    def run(self, sel, B: int, amp, slices: range | None = None, stream=None, accumulate=False,
            b_offset: int = 0, graph: bool = False):
        """Contract bitstrings [b_offset, b_offset + B) x ``slices``; writes (or
        adds, ``accumulate``) into ``amp[b_offset:b_offset + B]``.

        sel: dict node -> device int32 tensor of variant indices over the whole
        batch (None for single-variant sites); amp: device tensor of the engine
        dtype.  ``graph``: replay each chunk's launch sequence (projection, every
        step, slice sum) from a CUDA graph captured on the second call with the
        same buffers -- the path's launches then cost one graph launch (small,
        launch-bound networks such as configs[0]).
        """
        torch = self.torch
        plan = self.plan
        slices = range(plan.slice_count) if slices is None else slices
        if len(slices) == 0:
            return amp
        L = NV.lib()
        st = torch.cuda.current_stream(self.device) if stream is None else stream
        sptr = C.c_void_p(st.cuda_stream)
        pd = self._pd
        q0 = plan.path[0]
        for ci, (b0, nb, s0, ns) in enumerate(self.chunks(B, slices)):
            b0 += b_offset
            key = None
            if graph:
                acc_flag = 1 if (accumulate or s0 != slices.start) else 0
                key = (b0, nb, s0, ns, acc_flag, amp.data_ptr(),
                       tuple(self._selptr(sel, q, b0) for q in plan.path),
                       None if self._buf is None else self._buf[0].data_ptr())
                g = self._graphs.get(key)
                if g is not None:                  # replay: the descriptors are baked in
                    with torch.cuda.stream(st):
                        g.replay()
                    continue
            z = nb * ns
            bufa, bufb = self._buffers(z)
            cur, nxt = bufa, bufb
            f = pd.first
            f.Z, f.slices_per_b, f.s0 = z, ns, s0
            f.site.sel = self._selptr(sel, q0, b0)
            f.out = cur.data_ptr()
            f.out_zstride = prod(plan.first_dims) if plan.first_dims else 1
            for i, sp in enumerate(plan.steps):
                d = self._steps[i]
                d.Z, d.slices_per_b, d.s0 = z, ns, s0
                d.acc = cur.data_ptr()
                d.acc_zstride = sp.M * sp.K
                d.out = nxt.data_ptr()
                d.out_zstride = sp.M * sp.N
                d.site.sel = self._selptr(sel, sp.node, b0)
                cur, nxt = nxt, cur
            r = pd.reduce
            r.accumulate = 1 if (accumulate or s0 != slices.start) else 0
            r.B = nb
            r.slices_per_b = ns
            r.x = cur.data_ptr()
            r.x_zstride = 1
            r.amp = amp.data_ptr() + b0 * self.itemsize
            if graph:
                if key in self._graph_seen:
                    # capture on a side stream; the eager first call already set
                    # kernel attributes and warmed the allocator
                    g = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(g):
                        cs = torch.cuda.current_stream(self.device)
                        NV.check(L.tnc_contract_path(C.byref(pd), C.c_void_p(cs.cuda_stream)), "tnc_contract_path")
                    self._graphs[key] = g
                    with torch.cuda.stream(st):
                        g.replay()
                    continue
                self._graph_seen.add(key)
            NV.check(L.tnc_contract_path(C.byref(pd), sptr), "tnc_contract_path")
        return amp

    def _selptr(self, sel, q, b0):
        if sel is None or self.nvar[q] == 1:
            return None
        t = sel[q]
        return t.data_ptr() + 4 * b0

    def launches_per_chunk(self) -> int:
        return 2 + len(self.plan.steps)


def contract_pair_device(ta, a_dims, tb, b_dims, pairs, out_perm=None, conj_b=False,
                         batch: int = 1, a_zstride: int = 0, b_zstride: int = 0):
    """Batched pairwise contraction of device tensors through ``tnc_contract_pair``.

    ``ta`` / ``tb`` are contiguous complex CUDA tensors holding ``batch`` (or one
    broadcast, z-stride 0) row-major operands of shape ``a_dims`` / ``b_dims``.
    Returns a [batch, prod(out dims)] tensor; result axes are the unpaired axes
    of a then of b, permuted by ``out_perm``.
    """
    import torch

    NV.require_device()
    L = NV.lib()
    if ta.dtype != tb.dtype:
        raise EngineError("operand dtypes differ")
    code = NV.C64 if ta.dtype == torch.complex64 else NV.C128
    dev = ta.device
    adims = np.array(a_dims, dtype=np.int64)
    bdims = np.array(b_dims, dtype=np.int64)
    pa = np.array([p[0] for p in pairs], dtype=np.int32)
    pb = np.array([p[1] for p in pairs], dtype=np.int32)
    fa = [i for i in range(len(a_dims)) if i not in set(pa.tolist())]
    fb = [i for i in range(len(b_dims)) if i not in set(pb.tolist())]
    odims = [int(a_dims[i]) for i in fa] + [int(b_dims[i]) for i in fb]
    perm = list(range(len(odims))) if out_perm is None else list(out_perm)
    nout = prod(odims) if odims else 1
    out = torch.empty((batch, nout), dtype=ta.dtype, device=dev)
    ws_bytes = L.tnc_contract_pair_workspace(len(a_dims), adims.ctypes.data, len(b_dims), bdims.ctypes.data,
                                             len(pairs), pa.ctypes.data, pb.ctypes.data)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
    permarr = np.array(perm if perm else [0], dtype=np.int32)
    stream = torch.cuda.current_stream(dev).cuda_stream
    NV.check(L.tnc_contract_pair(code, batch, ta.data_ptr(), len(a_dims), adims.ctypes.data, a_zstride,
                                 tb.data_ptr(), len(b_dims), bdims.ctypes.data, b_zstride,
                                 len(pairs), pa.ctypes.data, pb.ctypes.data,
                                 permarr.ctypes.data if perm else None,
                                 1 if conj_b else 0, out.data_ptr(), nout, ws.data_ptr(), ws_bytes,
                                 C.c_void_p(stream)), "tnc_contract_pair")
    return out


def device_contract_pair(a: np.ndarray, b: np.ndarray, pairs, out_perm=None, conj_b=False,
                         dtype: str = "complex128") -> np.ndarray:
    """Host-array convenience wrapper of ``contract_pair_device`` (batch 1)."""
    import torch

    NV.require_device()
    tdt = torch.complex64 if dtype_code(dtype) == NV.C64 else torch.complex128
    dev = torch.device("cuda", torch.cuda.current_device())
    ta = torch.from_numpy(np.ascontiguousarray(a, dtype=np.complex128)).to(dev, tdt)
    tb = torch.from_numpy(np.ascontiguousarray(b, dtype=np.complex128)).to(dev, tdt)
    out = contract_pair_device(ta, a.shape, tb, b.shape, pairs, out_perm, conj_b)
    pset_a = {p[0] for p in pairs}
    pset_b = {p[1] for p in pairs}
    odims = [a.shape[i] for i in range(a.ndim) if i not in pset_a] + [b.shape[i] for i in range(b.ndim) if i not in pset_b]
    if out_perm is not None:
        odims = [odims[p] for p in out_perm]
    res = out[0].cpu().numpy().astype(np.complex128)
    return res.reshape(odims)


class PairPlan:
    """Reusable batched pairwise contraction (``tnc_pair_plan``): the layout
    analysis and offset tables are built once; each call launches only the
    kernel (asynchronously on the current stream)."""

    def __init__(self, a_dims, b_dims, pairs, dtype: str = "complex64", out_perm=None, conj_b=False):
        NV.require_device()
        self.L = NV.lib()
        self.code = dtype_code(dtype)
        self.a_dims = [int(d) for d in a_dims]
        self.b_dims = [int(d) for d in b_dims]
        self.pairs = [tuple(p) for p in pairs]
        adims = np.array(self.a_dims, dtype=np.int64)
        bdims = np.array(self.b_dims, dtype=np.int64)
        pa = np.array([p[0] for p in self.pairs], dtype=np.int32)
        pb = np.array([p[1] for p in self.pairs], dtype=np.int32)
        sa, sb = {p[0] for p in self.pairs}, {p[1] for p in self.pairs}
        odims = [d for i, d in enumerate(self.a_dims) if i not in sa] + [d for i, d in enumerate(self.b_dims) if i not in sb]
        perm = None
        if out_perm is not None:
            perm = np.array(list(out_perm), dtype=np.int32)
            odims = [odims[p] for p in out_perm]
        self.out_dims = odims
        self.K = prod(self.a_dims[p[0]] for p in self.pairs) if self.pairs else 1
        self.N = prod(d for i, d in enumerate(self.b_dims) if i not in sb)
        h = C.c_void_p()
        NV.check(self.L.tnc_pair_plan_create(self.code, len(adims), adims.ctypes.data, len(bdims), bdims.ctypes.data,
                                             len(pa), pa.ctypes.data if len(pa) else None,
                                             pb.ctypes.data if len(pb) else None,
                                             perm.ctypes.data if perm is not None else None,
                                             1 if conj_b else 0, C.byref(h)), "tnc_pair_plan_create")
        self._h = h

    @property
    def kernel(self) -> str:
        k = self.L.tnc_pair_plan_kernel(self._h)
        if k == NV.K_TC:
            # 3xTF32 by default; TNC_TC_F16=1 selects the fp16-split operands
            # (kind::f16) at K = 16 when the raw ring stages whole tiles (launch_tc)
            f16 = self.K == 16 and os.environ.get("TNC_TC_F16", "").startswith("1")
            return "tcgen05-3xfp16" if f16 else "tcgen05-3xtf32"
        return {NV.K_SKINNY: "tiled-permute", NV.K_GENERIC: "generic"}.get(k, str(k))

    def __call__(self, a, b, out, batch: int, a_zstride: int, b_zstride: int, out_zstride: int, stream=None):
        import torch

        st = torch.cuda.current_stream() if stream is None else stream
        NV.check(self.L.tnc_pair_plan_execute(self._h, batch, a.data_ptr(), a_zstride, b.data_ptr(), b_zstride,
                                              out.data_ptr(), out_zstride, C.c_void_p(st.cuda_stream)),
                 "tnc_pair_plan_execute")
        return out

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                self.L.tnc_pair_plan_destroy(h)
            except Exception:
                pass
            self._h = None


def project_variants(variants, bits, out, K_times_N: int, stream=None):
    """Bitstring projection of a site: out[b] = variants[bits[b]] (tnc_project
    gather).  variants: device [V, K*N]; bits: device int32 [B]."""
    import torch

    L = NV.lib()
    code = NV.C64 if variants.dtype == torch.complex64 else NV.C128
    d = NV.ProjectDesc()
    d.dtype = code
    d.conj = 0
    d.Z = int(bits.numel())
    d.slices_per_b = 1
    d.s0 = 0
    _fill_site(d.site, variants.data_ptr(), K_times_N, [])
    d.site.sel = bits.data_ptr()
    d.out = out.data_ptr()
    d.out_zstride = K_times_N
    d.nd = 1
    d.dim[0] = K_times_N
    d.src_stride[0] = 1
    st = torch.cuda.current_stream() if stream is None else stream
    NV.check(L.tnc_project(C.byref(d), C.c_void_p(st.cuda_stream)), "tnc_project")
    return out
