"""Torch-facing API over the C ABI (same names as include/chem.h).

PyTorch provides device memory and the current CUDA stream; every computation happens in
libchem.so.  Arrays follow the C ABI layout: per-cell scalars are 1-D float64 CUDA tensors of
length >= n, species arrays are [ns, ld] float64 CUDA tensors (component-major).
"""
from __future__ import annotations

import ctypes
import dataclasses

import numpy as np
import torch

from . import binding as _b
from . import mechanism as _mech


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def _check(t, name, dtype=torch.float64, n=None, device=None):
    """The C ABI cannot see a tensor's dtype, device or length: this binding is the only guard
    against a kernel reading or writing past a buffer (or a host pointer used as a device one)."""
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor (there is no CPU path)")
    if t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}")
    if device is not None and t.device != device:
        raise ValueError(f"{name} is on {t.device}, the ctx on {device}")
    if n is not None:
        if t.dim() != 1 or (t.numel() > 1 and t.stride(0) != 1) or t.numel() < n:
            raise ValueError(f"{name} must be a contiguous 1-D tensor of >= {n} elements")


def _species(Y, ns, n=None):
    _check(Y, "Y")
    if Y.dim() != 2 or Y.shape[0] != ns or (Y.shape[1] > 1 and Y.stride(1) != 1):
        raise ValueError(f"Y must be [ns={ns}, ld] with unit stride along cells")
    if n is not None and Y.shape[1] < n:
        raise ValueError(f"Y has {Y.shape[1]} cells, the call {n}")
    if n is not None and Y.shape[0] > 1 and Y.stride(0) < n:
        raise ValueError("Y's component stride (ld) is smaller than the cell count")
    return Y.stride(0)


@dataclasses.dataclass
class Box:
    """One AMR box (FAB analogue): views into caller tensors, integrated in place."""
    rho: torch.Tensor
    e: torch.Tensor
    T: torch.Tensor
    Y: torch.Tensor          # [ns, ld]
    dt: float
    solid: torch.Tensor | None = None

    @property
    def ncells(self):
        return self.rho.shape[0]


class Chem:
    """A chem_ctx bound to one mechanism and one CUDA device."""

    def __init__(self, mech="h2air_li2004", device=None, **opts):
        self.lib = _b.load_library()
        self.mech = mech if isinstance(mech, _mech.MechTables) else _mech.load(mech)
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        self.ns = self.mech.ns
        desc, self._keep = _b.mech_desc(self.mech)
        self.opts = _b.default_opts(self.lib)
        self._set(opts)
        h = ctypes.c_void_p()
        rc = self.lib.chem_init(ctypes.byref(desc), ctypes.byref(self.opts), self.device.index, ctypes.byref(h))
        if rc != 0:
            raise _b.ChemError(rc, self.lib)
        self._h = h
        self._ws = None
        self._ws_layout = {}
        self.last_stats = None

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            self.lib.chem_finalize(h)
            self._h = None

    @property
    def structure(self) -> str:
        return self.lib.chem_structure_name(self._h).decode()

    def _set(self, opts):
        names = {f for f, _ in _b.ChemOpts._fields_}
        for k, v in opts.items():
            if k not in names:       # ctypes would silently add a Python attribute
                raise TypeError(f"unknown chem_opts field {k!r}")
            setattr(self.opts, k, v)

    def set_opts(self, **opts):
        self._set(opts)
        rc = self.lib.chem_set_opts(self._h, ctypes.byref(self.opts))
        if rc != 0:
            raise _b.ChemError(rc, self.lib)

    def set_trace(self, rows, nboxes):
        """Enable the App. B activity trace: returns the device int32 [rows, nboxes] tensor that the
        next integrate calls fill (row 0 after the gate, row i after bulk launch i)."""
        if rows <= 0:
            self._trace = None
            self._call(self.lib.chem_set_trace(self._h, None, 0))
            return None
        self._trace = torch.zeros((rows, nboxes), dtype=torch.int32, device=self.device)
        self._call(self.lib.chem_set_trace(self._h, _ptr(self._trace), rows))
        return self._trace

    def _stream(self):
        return ctypes.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)

    def _call(self, rc):
        if rc != 0:
            raise _b.ChemError(rc, self.lib)

    def workspace(self, max_cells, max_boxes=1, layout=None):
        """Device workspace for a call (~45 B/cell).  `layout` (a hashable key of the call's cell
        layout: cell count, box count, first rho pointer) selects a workspace of its own, so the
        per-cell cost hints the heavy-first schedule reads survive between calls
        on that layout when calls on other layouts (AMR levels) interleave.  At most 8 layouts are
        kept (least recently used dropped): a caller that allocates fresh state tensors every step
        makes a new layout each call, so it should call release_workspaces() or keep its tensors."""
        nbytes = self.lib.chem_workspace_bytes(self._h, int(max_cells), int(max_boxes))
        if layout is None:
            if self._ws is None or self._ws.numel() < nbytes:
                self._ws = torch.zeros(max(nbytes, 1), dtype=torch.uint8, device=self.device)
            return self._ws
        ws = self._ws_layout.pop(layout, None)
        if ws is None or ws.numel() < nbytes:
            ws = torch.zeros(max(nbytes, 1), dtype=torch.uint8, device=self.device)
        self._ws_layout[layout] = ws            # most recently used last
        while len(self._ws_layout) > 8:
            self._ws_layout.pop(next(iter(self._ws_layout)))
        self._ws = ws
        return ws

    def release_workspaces(self):
        self._ws = None
        self._ws_layout.clear()

    def forget_hints(self):
        """Zero every cached workspace: the next call of each layout runs as a layout's first call
        (no cost hints; Alg. 3's bulk-sparse schedule).  Enqueued on the current stream."""
        for ws in self._ws_layout.values():
            ws.zero_()
        if self._ws is not None:
            self._ws.zero_()

    def _cells(self, n, Y, **scalars):
        ld = _species(Y, self.ns, n)
        if Y.device != self.device:
            raise ValueError(f"Y is on {Y.device}, the ctx on {self.device}")
        for nm, t in scalars.items():
            _check(t, nm, n=n, device=self.device)
        return ld

    # ---- point evaluations ---------------------------------------------------------------
    def rates(self, rho, T, Y, out=None):
        n = rho.shape[0]
        ld = self._cells(n, Y, rho=rho, T=T)
        if out is None:
            out = torch.empty((self.ns, ld), dtype=torch.float64, device=self.device)
        elif out.shape[0] != self.ns or out.stride(0) != ld or out.stride(1) != 1:
            raise ValueError("out must be [ns, ld] with Y's ld")
        self._call(self.lib.chem_rates(self._h, n, ld, _ptr(rho), _ptr(T), _ptr(Y), _ptr(out), self._stream()))
        return out

    def rhs(self, rho, T, Y, out=None):
        n = rho.shape[0]
        ld = self._cells(n, Y, rho=rho, T=T)
        if out is not None and (out.shape[0] != self.ns + 1 or out.stride(0) != ld or out.stride(1) != 1):
            raise ValueError("out must be [ns + 1, ld] with Y's ld")
        if out is None:
            out = torch.empty((self.ns + 1, ld), dtype=torch.float64, device=self.device)
        self._call(self.lib.chem_rhs(self._h, n, ld, _ptr(rho), _ptr(T), _ptr(Y), _ptr(out), self._stream()))
        return out

    def jacobian(self, rho, T, Y):
        n = rho.shape[0]
        ld = self._cells(n, Y, rho=rho, T=T)
        nn = self.ns + 1
        J = torch.empty((nn * nn, ld), dtype=torch.float64, device=self.device)
        self._call(self.lib.chem_jacobian(self._h, n, ld, _ptr(rho), _ptr(T), _ptr(Y), _ptr(J), self._stream()))
        return J.view(nn, nn, ld)

    def temperature(self, e, Y, T):
        """In place: T <- Newton(e, Y) seeded with T."""
        n = e.shape[0]
        ld = self._cells(n, Y, e=e, T=T)
        self._call(self.lib.chem_temperature(self._h, n, ld, _ptr(e), _ptr(Y), _ptr(T), self._stream()))
        return T

    def internal_energy(self, U, out=None):
        """Alg. 1: e = rho E/rho - |u|^2/2 from conserved U [5, ld] (component-major)."""
        _check(U, "U")
        if U.dim() != 2 or U.shape[0] != 5 or U.stride(1) != 1:
            raise ValueError("U must be [5, ld]: rho, rho ux, rho uy, rho uz, rho E")
        n = U.shape[1]
        if out is None:
            out = torch.empty(n, dtype=torch.float64, device=self.device)
        self._call(self.lib.chem_internal_energy(self._h, n, U.stride(0), _ptr(U), _ptr(out), self._stream()))
        return out

    def strang_half_step(self, boxes, dt_flow, rtol=1e-9, atol=1e-20, box_cost=None):
        """Chemistry half of a Strang-split flow step: integrate every box over dt_flow/2.
        A flow solver calls this before and after its own dt_flow update."""
        half = [Box(b.rho, b.e, b.T, b.Y, 0.5 * dt_flow, b.solid) for b in boxes]
        return self.integrate_boxes(half, rtol=rtol, atol=atol, box_cost=box_cost)

    def energy(self, T, Y, out=None):
        n = T.shape[0]
        ld = self._cells(n, Y, T=T)
        if out is not None:
            _check(out, "out", n=n, device=self.device)
        if out is None:
            out = torch.empty(n, dtype=torch.float64, device=self.device)
        self._call(self.lib.chem_energy(self._h, n, ld, _ptr(T), _ptr(Y), _ptr(out), self._stream()))
        return out

    # ---- integration ------------------------------------------------------------------------
    def integrate(self, rho, e, T, Y, dt, rtol=1e-9, atol=1e-20, solid=None):
        """In place on T and Y (chem_integrate).  Returns the chem_stats dict."""
        n = rho.shape[0]
        ld = self._cells(n, Y, rho=rho, e=e, T=T)
        if solid is not None:
            _check(solid, "solid", torch.uint8, n=n, device=self.device)
        ws = self.workspace(n, 1, layout=(n, 1, rho.data_ptr()))
        st = _b.ChemStats()
        self._call(self.lib.chem_integrate(self._h, n, ld, _ptr(rho), _ptr(e), _ptr(T), _ptr(Y), _ptr(solid),
                                           float(dt), float(rtol), float(atol), _ptr(ws), ws.numel(),
                                           ctypes.byref(st), self._stream()))
        self.last_stats = st.to_dict()
        return self.last_stats

    def integrate_boxes(self, boxes, rtol=1e-9, atol=1e-20, box_cost=None):
        """Fused multi-box call (chem_integrate_boxes).  box_cost: optional float64 CUDA [nboxes]."""
        nb = len(boxes)
        arr = (_b.ChemBox * nb)()
        total = 0
        if nb < 1:
            raise ValueError("integrate_boxes needs at least one box")
        for i, bx in enumerate(boxes):
            ld = self._cells(bx.ncells, bx.Y, rho=bx.rho, e=bx.e, T=bx.T)
            if bx.solid is not None:
                _check(bx.solid, "solid", torch.uint8, n=bx.ncells, device=self.device)
            arr[i].rho = bx.rho.data_ptr()
            arr[i].e = bx.e.data_ptr()
            arr[i].T = bx.T.data_ptr()
            arr[i].Y = bx.Y.data_ptr()
            arr[i].solid = bx.solid.data_ptr() if bx.solid is not None else None
            arr[i].ncells = bx.ncells
            arr[i].ld = ld
            arr[i].dt = float(bx.dt)
            total += bx.ncells
        ws = self.workspace(total, nb, layout=(total, nb, boxes[0].rho.data_ptr()))
        if box_cost is not None:
            _check(box_cost, "box_cost", n=nb, device=self.device)
        st = _b.ChemStats()
        self._call(self.lib.chem_integrate_boxes(self._h, nb, arr, float(rtol), float(atol), _ptr(ws), ws.numel(),
                                                 _ptr(box_cost), ctypes.byref(st), self._stream()))
        self.last_stats = st.to_dict()
        return self.last_stats

    def box_active(self, boxes):
        """int32 CUDA tensor [nboxes]: cells of each box the gate would integrate (chem_box_active; reads
        only T and solid)."""
        nb = len(boxes)
        arr = (_b.ChemBox * nb)()
        for i, bx in enumerate(boxes):
            _check(bx.T, "T", n=bx.ncells, device=self.device)
            if bx.solid is not None:
                _check(bx.solid, "solid", torch.uint8, n=bx.ncells, device=self.device)
            arr[i].T = bx.T.data_ptr()
            arr[i].solid = bx.solid.data_ptr() if bx.solid is not None else None
            arr[i].ncells = bx.ncells
            arr[i].ld = bx.ncells
            arr[i].dt = float(bx.dt) if bx.dt > 0 else 1.0
        nbytes = self.lib.chem_workspace_bytes(self._h, 0, nb)
        if getattr(self, "_ws_small", None) is None or self._ws_small.numel() < nbytes:
            self._ws_small = torch.zeros(max(nbytes, 1), dtype=torch.uint8, device=self.device)
        out = torch.empty(nb, dtype=torch.int32, device=self.device)
        self._call(self.lib.chem_box_active(self._h, nb, arr, _ptr(out), _ptr(self._ws_small), self._ws_small.numel(),
                                            self._stream()))
        return out

    def cell_status(self, n=None, first=0, substeps=False):
        """int8 CUDA tensor of CHEM_CELL_* codes for global cells [first, first + n) of
        the last integrate / integrate_boxes call (boxes numbered in call order); with
        substeps=True also the int32 per-cell attempted substeps of that call."""
        ws = self._ws
        if ws is None:
            raise RuntimeError("no integrate call yet")
        if n is None:
            n = self.last_stats["cells"] - first
        out = torch.empty(max(n, 0), dtype=torch.int8, device=self.device)
        k = torch.empty(max(n, 0), dtype=torch.int32, device=self.device) if substeps else None
        self._call(self.lib.chem_cell_status(self._h, _ptr(ws), ws.numel(), int(first), int(n), _ptr(out),
                                             _ptr(k), self._stream()))
        return (out, k) if substeps else out


class HostRunner:
    """End-to-end public-API path for host-resident data (the bench's `e2e` leg): pinned host
    buffers -> H2D copies -> chem_integrate_boxes -> D2H of (T, Y), in place on the host like the
    device API: each group's pinned slab [rho_*][e_*][T_*][Y_*] goes to the device and its [T_*][Y_*]
    results come back into the same slab.  Gated cells are never read or written, so
    only boxes the step touched (box_cost > 0) are copied back - an untouched box's host T, Y are
    already its outputs - and, on the unpipelined path, every box's T goes over first and rho, e, Y
    follow only for boxes the gate finds active (chem_box_active).

    With a single fused call per step, the boxes are processed in `chunks` groups through three
    CUDA streams so that the H2D copy of group i+1 and the D2H copy of group i-1 run on the copy
    engines while group i integrates (the host blocks inside chem_integrate_boxes only on the
    compute stream's counters, which the library reads through mapped memory, not a copy engine);
    a pipelined group returns the results of all its boxes."""

    def __init__(self, chem: Chem, host_boxes, calls=None, chunks=4, selective=True, taper=2.0):
        self.chem = chem
        self.selective = selective      # unpipelined path: H2D of rho, e, Y only for boxes with active cells
        self.calls = calls or [list(range(len(host_boxes)))]
        dev = chem.device
        nb = len(host_boxes)
        self.pipelined = len(self.calls) == 1 and len(self.calls[0]) >= chunks > 1
        if self.pipelined:
            # tapered groups: the first group's H2D and the last group's D2H are the copies nothing
            # overlaps, so those two groups get 1/taper of the share of the middle ones
            ids = self.calls[0]
            w = [1.0] + [float(taper)] * (chunks - 2) + [1.0] if chunks > 2 else [1.0] * chunks
            cuts = np.round(np.cumsum([0.0] + w) / sum(w) * len(ids)).astype(int)
            self.groups = [ids[cuts[g]:cuts[g + 1]] for g in range(chunks) if cuts[g + 1] > cuts[g]]
            self.s_h2d = torch.cuda.Stream(dev)
            self.s_d2h = torch.cuda.Stream(dev)
        else:
            self.groups = [list(range(nb))]
        self.dev_boxes = [None] * nb
        self.out_T, self.out_Y = [None] * nb, [None] * nb
        self.ranges = [None] * nb          # per box: (group, T offset, n, Y offset, ns * n) in the slab
        self.slabs = []
        for g, grp in enumerate(self.groups):
            n = [host_boxes[i]["rho"].numel() for i in grp]
            ns = [host_boxes[i]["Y"].shape[0] for i in grp]
            tot = sum(n)
            size = 3 * tot + sum(a * c for a, c in zip(n, ns))
            h = torch.empty(size, dtype=torch.float64).pin_memory()
            d = torch.empty(size, dtype=torch.float64, device=dev)
            o = [0, tot, 2 * tot, 3 * tot]   # rho, e, T, Y cursors
            for i, ni, si in zip(grp, n, ns):
                self.dev_boxes[i] = Box(d[o[0]:o[0] + ni], d[o[1]:o[1] + ni], d[o[2]:o[2] + ni],
                                        d[o[3]:o[3] + ni * si].view(si, ni), host_boxes[i]["dt"])
                self.out_T[i] = h[o[2]:o[2] + ni]
                self.out_Y[i] = h[o[3]:o[3] + ni * si].view(si, ni)
                self.ranges[i] = (g, o[2], ni, o[3], ni * si)
                o = [o[0] + ni, o[1] + ni, o[2] + ni, o[3] + ni * si]
            self.slabs.append((h, d, 2 * tot))
        self.load_inputs(host_boxes)
        self.h2d_bytes_full = sum(s_[0].numel() * 8 for s_ in self.slabs)
        self.h2d_bytes = self.h2d_bytes_full   # of the last step
        self.d2h_bytes_full = sum((s_[0].numel() - s_[2]) * 8 for s_ in self.slabs)
        self.d2h_bytes = 0                  # of the last step (touched boxes only)

    def load_inputs(self, host_boxes):
        """Copy new host inputs (same shapes as at construction) into the pinned slabs (host memcpy;
        the next step() moves them).  Needed before every step whose inputs are not the previous
        step's outputs (the slabs are updated in place)."""
        torch.cuda.synchronize(self.chem.device)    # the last step's D2H writes these slabs
        for g, grp in enumerate(self.groups):
            h = self.slabs[g][0]
            tot = sum(host_boxes[i]["rho"].numel() for i in grp)
            o = [0, tot, 2 * tot, 3 * tot]
            for i in grp:
                hb = host_boxes[i]
                ni, si = hb["rho"].numel(), hb["Y"].shape[0]
                h[o[0]:o[0] + ni].copy_(hb["rho"].reshape(-1))
                h[o[1]:o[1] + ni].copy_(hb["e"].reshape(-1))
                h[o[2]:o[2] + ni].copy_(hb["T"].reshape(-1))
                h[o[3]:o[3] + ni * si].copy_(hb["Y"].reshape(-1))
                o = [o[0] + ni, o[1] + ni, o[2] + ni, o[3] + ni * si]

    def _h2d_group(self, g):
        h, d, _ = self.slabs[g]
        d.copy_(h, non_blocking=True)

    def _h2d_full(self, g):
        self._h2d_group(g)
        return self.slabs[g][0].numel() * 8

    def _d2h_boxes(self, boxes):
        """D2H of the [T][Y] results of `boxes` into their slabs: one copy per group when every box
        of the group is touched, else two per touched box."""
        by_group = {}
        for i in boxes:
            by_group.setdefault(self.ranges[i][0], []).append(i)
        nbytes = 0
        for g, ids in by_group.items():
            h, d, t0 = self.slabs[g]
            if len(ids) == len(self.groups[g]):
                h[t0:].copy_(d[t0:], non_blocking=True)
                nbytes += (h.numel() - t0) * 8
                continue
            for i in ids:
                _, to, n, yo, ny = self.ranges[i]
                h[to:to + n].copy_(d[to:to + n], non_blocking=True)
                h[yo:yo + ny].copy_(d[yo:yo + ny], non_blocking=True)
                nbytes += (n + ny) * 8
        return nbytes

    def _call(self, ids, rtol, atol, touched_only=True):
        if not touched_only:
            # pipelined groups: every box's results come back.  Reading box_cost here would put a
            # copy-engine D2H on the compute stream, and the next call's commands would then wait for
            # the group D2H queued meanwhile on the copy stream (tools/e2e_timeline.py)
            st = self.chem.integrate_boxes([self.dev_boxes[i] for i in ids], rtol=rtol, atol=atol)
            return st, list(ids)
        cost = torch.zeros(len(ids), dtype=torch.float64, device=self.chem.device)
        st = self.chem.integrate_boxes([self.dev_boxes[i] for i in ids], rtol=rtol, atol=atol, box_cost=cost)
        touched = [i for i, c in zip(ids, cost.cpu().tolist()) if c > 0]   # the call has synchronised
        return st, touched

    def _h2d_active(self, g):
        """Selective H2D of group g: every box's T first, then rho, e and Y only of the boxes whose gate
        finds active cells (chem_box_active) - the kernels never read a gated cell's rho, e or Y."""
        h, d, t0 = self.slabs[g]
        tot = t0 // 2
        d[2 * tot:3 * tot].copy_(h[2 * tot:3 * tot], non_blocking=True)
        grp = self.groups[g]
        act = self.box_active([self.dev_boxes[i] for i in grp])
        nbytes = tot * 8
        if all(a > 0 for a in act):
            d[:2 * tot].copy_(h[:2 * tot], non_blocking=True)
            d[3 * tot:].copy_(h[3 * tot:], non_blocking=True)
            return nbytes + (h.numel() - tot) * 8
        for i, a in zip(grp, act):
            if a > 0:
                _, to, n, yo, ny = self.ranges[i]
                ro, eo = to - 2 * tot, to - tot
                d[ro:ro + n].copy_(h[ro:ro + n], non_blocking=True)
                d[eo:eo + n].copy_(h[eo:eo + n], non_blocking=True)
                d[yo:yo + ny].copy_(h[yo:yo + ny], non_blocking=True)
                nbytes += (2 * n + ny) * 8
        return nbytes

    def box_active(self, boxes):
        return self.chem.box_active(boxes).cpu().tolist()

    def step(self, rtol, atol):
        if not self.pipelined:
            self.h2d_bytes = self._h2d_active(0) if self.selective else self._h2d_full(0)
            st, touched = [], set()
            for c in self.calls:
                s_, t_ = self._call(c, rtol, atol)
                st.append(s_)
                touched.update(t_)
            self.d2h_bytes = self._d2h_boxes(sorted(touched))
            return st
        comp = torch.cuda.current_stream(self.chem.device)
        ev_in = [torch.cuda.Event() for _ in self.groups]
        st = []
        nbytes = 0
        with torch.cuda.stream(self.s_h2d):
            self.s_h2d.wait_stream(comp)            # the previous step's D2H reads must not be overwritten early
            self.s_h2d.wait_stream(self.s_d2h)
            self._h2d_group(0)
            ev_in[0].record(self.s_h2d)
        for g, idx in enumerate(self.groups):
            if g + 1 < len(self.groups):
                with torch.cuda.stream(self.s_h2d):
                    self._h2d_group(g + 1)
                    ev_in[g + 1].record(self.s_h2d)
            comp.wait_event(ev_in[g])
            s_, touched = self._call(idx, rtol, atol, touched_only=False)
            st.append(s_)
            done = torch.cuda.Event()
            done.record(comp)
            with torch.cuda.stream(self.s_d2h):
                self.s_d2h.wait_event(done)
                nbytes += self._d2h_boxes(touched)
        comp.wait_stream(self.s_d2h)                # the step ends when the last result is on the host
        self.d2h_bytes = nbytes
        return st


def activity_lines(trace, boxes, levels=None, t=0.0, kmax=5):
    """Format an activity trace in the paper's App. B line format:
    'Level <level>, FAB <fab_ID>, t = <time>, step = <iteration>, n_cells = <total>, n_active = <active>'
    (step = attempted-substep budget consumed: K_max per bulk launch)."""
    tr = trace.cpu().numpy()
    out = []
    for b, bx in enumerate(boxes):
        lv = 0 if levels is None else levels[b]
        for it in range(tr.shape[0]):
            out.append(f"Level {lv}, FAB {b}, t = {t:g}, step = {it * kmax}, n_cells = {bx.ncells}, "
                       f"n_active = {int(tr[it, b])}")
    return out
