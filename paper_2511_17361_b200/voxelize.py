"""The voxelize module of SPEC.md:317-400, on B200 kernels.

Drop-in operations (same names, arguments and meaning as the SPEC):

- ``voxelize(scene, spec, cfg) -> (SemanticGrid, DenseGrids)``
- ``voxelize_bruteforce(scene, spec, cfg) -> (SemanticGrid, DenseGrids)`` SPEC.md:355-363
- ``finalize(dense, tau, classes) -> SemanticGrid``
- types ``VoxelGridSpec`` / ``VoxelizeConfig`` / ``DenseGrids`` / ``SemanticGrid``
  

plus the throughput entry the scene-per-call API cannot provide:

- ``Voxelizer(spec, cfg, n_classes)(batch)`` — F frames of N primitives
  (``PrimitiveBatch``, FP64 SoA on host or device) in one call, outputs left
  on the device as torch tensors.

Everything runs in libsqv.so (include/sqv.h ``sqv_voxelize``): prep ->
scan -> emit -> radix sort -> evaluate+finalize.  There is no CPU path.

Layout: voxel arrays are x-fastest.  Device tensors are
``labels[F, nz, ny, nx]`` (uint8), ``v_o[F, nz, ny, nx]``,
``v_c[F, nz, ny, nx, C]`` (float32, SPEC.md:113 allows FP32 storage).  The
drop-in grids expose the SPEC's logical (nx, ny, nz) indexing as
transposed NumPy views of that memory.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import Any

import numpy as np

from . import _lib
from .core import ClassTable, PrimitiveBatch, Scene, bad_bits_message

SEMANTIC_MODES = ("logit-sum", "prob-sum")
PRECISIONS = ("fast", "strict")


@dataclass(frozen=True)
class VoxelGridSpec:
    """origin (min corner, m), dims (nx, ny, nz), resolution (m).  Occ3D default
    (SPEC.md:326): (-40, -40, -1), (200, 200, 16), 0.4."""

    origin: tuple = (-40.0, -40.0, -1.0)
    dims: tuple = (200, 200, 16)
    resolution: float = 0.4

    def __post_init__(self):
        origin = tuple(float(v) for v in self.origin)
        dims = tuple(int(v) for v in self.dims)
        if len(origin) != 3 or len(dims) != 3:
            raise ValueError("origin and dims must have 3 components")
        if not all(np.isfinite(origin)):
            raise ValueError("origin must be finite")
        if any(d < 1 for d in dims):
            raise ValueError("dims must be >= 1 each")
        if not (float(self.resolution) > 0.0 and np.isfinite(float(self.resolution))):
            raise ValueError("resolution must be > 0")
        object.__setattr__(self, "origin", origin)
        object.__setattr__(self, "dims", dims)
        object.__setattr__(self, "resolution", float(self.resolution))

    @property
    def n_voxels(self) -> int:
        return self.dims[0] * self.dims[1] * self.dims[2]

    def _c(self) -> _lib.Grid:
        g = _lib.Grid()
        g.origin[:] = self.origin
        g.dims[:] = self.dims
        g.resolution = self.resolution
        return g


@dataclass(frozen=True)
class VoxelizeConfig:
    """tau (default 0.01), neighborhood_radius (voxels, default 5),
    semantic_mode ("logit-sum" | "prob-sum").  window_extent is the ledger's
    max-K expansion factor (default 2.5).  precision selects the
    device numerics: "strict" (default; densities within 1e-5 relative down to
    1e-3*tau) or "fast" (all logs on the SFU, ~5% faster; 3e-5 relative down to
    1e-3*tau) — see DESIGN.md §Numerics."""

    tau: float = 0.01
    neighborhood_radius: int = 5
    semantic_mode: str = "logit-sum"
    window_extent: float = 2.5
    precision: str = "strict"

    def __post_init__(self):
        if not (float(self.tau) >= 0.0):
            raise ValueError("tau must be >= 0")
        if int(self.neighborhood_radius) != self.neighborhood_radius or self.neighborhood_radius < 0:
            raise ValueError("neighborhood_radius must be a non-negative integer")
        if self.semantic_mode not in SEMANTIC_MODES:
            raise ValueError(f"semantic_mode must be one of {SEMANTIC_MODES}")
        if not (float(self.window_extent) >= 0.0 and np.isfinite(float(self.window_extent))):
            raise ValueError("window_extent must be finite and >= 0")
        if self.precision not in PRECISIONS:
            raise ValueError(f"precision must be one of {PRECISIONS}")


@dataclass
class DenseGrids:
    """v_o (nx, ny, nz) >= 0 and v_c (nx, ny, nz, C).
    ``spec`` (optional) is the grid the arrays were voxelized on; voxelize()
    sets it and finalize() carries it into the SemanticGrid."""

    v_o: Any
    v_c: Any
    spec: Any = None


@dataclass
class SemanticGrid:
    """labels (nx, ny, nz): class id in [0, C) or classes.free_index."""

    labels: Any
    spec: VoxelGridSpec
    classes: ClassTable


@dataclass
class VoxelizeResult:
    """Device outputs of one batched call (torch tensors, x-fastest memory)."""

    labels: Any                 # uint8 [F, nz, ny, nx]; free voxels = free_code
    v_o: Any = None             # float32 [F, nz, ny, nx]
    v_c: Any = None             # float32 [F, nz, ny, nx, C]
    free_code: int = 255
    n_pairs: int = 0            # algorithmic (primitive, in-window voxel) pairs
    n_entries: int = 0          # (tile, primitive) bin entries
    bins: dict | None = None    # windows / tile_off / prim_ids when requested


def free_code_for(free_index: int, n_classes: int) -> int:
    """The u8 label written for free voxels: free_index itself when it fits a
    byte, else 255 (remapped on the host by ``SemanticGrid`` construction)."""
    if 0 <= free_index <= 255 and free_index >= n_classes:
        return int(free_index)
    return 255


class Voxelizer:
    """Reusable B200 voxelizer for one grid/config/class count.

    Holds the device workspace (grown on demand, torch caching allocator) and
    runs ``sqv_voxelize`` on the current CUDA stream.
    """

    def __init__(self, spec: VoxelGridSpec = VoxelGridSpec(), cfg: VoxelizeConfig = VoxelizeConfig(),
                 n_classes: int = 18, free_index: int | None = None, *, truncate: bool = True,
                 device=None):
        import torch
        self.torch = torch
        self.device = _lib.require_cuda(device)
        self.L = _lib.lib()
        if not (1 <= n_classes <= _lib.MAX_CLASSES):
            raise ValueError(f"n_classes must lie in [1, {_lib.MAX_CLASSES}] on the device path")
        self.spec, self.cfg, self.C = spec, cfg, int(n_classes)
        self.free_index = self.C if free_index is None else int(free_index)
        if 0 <= self.free_index < self.C:
            raise ValueError("free_index must lie outside [0, C)")
        self.free_code = free_code_for(self.free_index, self.C)
        self.truncate = bool(truncate)
        self._grid = spec._c()
        c = _lib.Cfg()
        c.tau = float(cfg.tau)
        c.neighborhood_radius = int(cfg.neighborhood_radius)
        c.truncate = int(self.truncate)
        c.semantic_mode = SEMANTIC_MODES.index(cfg.semantic_mode)
        c.free_label = self.free_code
        c.window_extent = float(cfg.window_extent)
        c.precision = PRECISIONS.index(cfg.precision)
        self._cfg = c
        self._ws = [None, None]  # one workspace per pipelined stream slot
        self.tiles_per_frame = int(self.L.sqv_tiles_per_frame(ctypes.byref(self._grid)))

    # ---- inputs -----------------------------------------------------------
    def _dev(self, a, dtype):
        t = self.torch
        if isinstance(a, np.ndarray):
            a = t.from_numpy(np.ascontiguousarray(a))
        a = a.to(device=self.device, dtype=dtype, non_blocking=True)
        return a.contiguous()

    def to_device(self, batch: PrimitiveBatch) -> PrimitiveBatch:
        t = self.torch
        f = [self._dev(getattr(batch, k), t.float64) for k in PrimitiveBatch.FIELDS]
        nv = None if batch.n_valid is None else self._dev(batch.n_valid, t.int32)
        return PrimitiveBatch(*f, n_valid=nv)

    def _workspace(self, nbytes: int, slot: int = 0):
        ws = self._ws[slot]
        if ws is None or ws.numel() < nbytes:
            # allocated on the stream that will use it (torch's allocator
            # keys blocks by stream)
            ws = self.torch.empty(int(nbytes * 1.25) + 4096, dtype=self.torch.uint8,
                                  device=self.device)
            self._ws[slot] = ws
        return ws

    def run_many(self, batches, outs, *, dense: bool = True, on_device=None):
        """Voxelize device-resident batches back to back on two alternating
        CUDA streams, so the per-batch binning (prep, the one header
        readback, emit, sort, masks) of batch k+1 overlaps the evaluation of
        batch k.  ``outs`` = two preallocated results (``alloc``), reused
        alternately; ``on_device(k, result)`` runs on batch k's stream right
        after it (e.g. confusion counts).  The caller's current stream waits
        for both streams on return (no host sync)."""
        t = self.torch
        cur = t.cuda.current_stream(self.device)
        if getattr(self, "_side", None) is None:
            self._side = t.cuda.Stream(self.device)
        streams = (cur, self._side)
        self._side.wait_stream(cur)
        for k, b in enumerate(batches):
            slot = k & 1
            with t.cuda.stream(streams[slot]):
                r = self(b, dense=dense, out=outs[slot], _slot=slot)
                if on_device is not None:
                    on_device(k, r)
        cur.wait_stream(self._side)

    # ---- pipelined host streams ----------------------------------------------
    def stream(self, batches, *, dense: bool = True, on_device=None, labels_out=None,
               edge_pieces: int = 4):
        """Voxelize a sequence of host batches (pinned torch tensors for real
        overlap) with copies overlapped: the H2D copy of batch k+1 and the D2H
        copy of batch k-1's labels run on two copy streams while batch k is
        evaluated; consecutive batches alternate two compute streams (the
        current one and a side stream, as in ``run_many``) so a batch's
        binning overlaps the previous evaluation.  Input slots and device
        label buffers are triple-buffered: batch k's binning waits only for
        copies that finished a whole batch earlier, so it is ready to run the
        moment batch k-2's evaluation ends (with double buffers it also waited
        for batch k-2's label D2H / batch k's H2D, issued only then, and lost
        its slot to batch k-1's evaluation).  The first and the last batch run
        as ``edge_pieces`` frame ranges (alternating the two compute streams
        too), so evaluation starts after the first range's H2D copy and only
        the last range's labels are copied after the final evaluation: the
        pipeline fills and drains at a quarter of a batch.  (Per-frame
        results depend on the frame grouping only through the evaluator's
        density-based kernel choice, see sqv_eval_tc_impl.cuh launch_tc.)
        ``on_device(k, result)`` is called once per batch, on its compute
        stream, after all of it (e.g. confusion counts).
        Returns the host label tensors [F, nz, ny, nx] (uint8, pinned), valid
        when this call returns."""
        t = self.torch
        nx, ny, nz = self.spec.dims
        comp0 = t.cuda.current_stream(self.device)
        if getattr(self, "_side", None) is None:
            self._side = t.cuda.Stream(self.device)
        comps = (comp0, self._side)
        self._side.wait_stream(comp0)
        h2d, d2h = t.cuda.Stream(self.device), t.cuda.Stream(self.device)
        nb = len(batches)
        if nb == 0:
            return []
        host = [{k: (getattr(b, k) if isinstance(getattr(b, k), t.Tensor)
                     else t.from_numpy(np.ascontiguousarray(getattr(b, k))))
                 for k in PrimitiveBatch.FIELDS} for b in batches]
        shapes = {k: (tuple(v.shape), v.dtype) for k, v in host[0].items()}
        F = batches[0].n_frames
        # input slots / device label buffers; the same allocations for any
        # number of batches, so the caching allocator reuses the previous
        # call's blocks (a different pattern makes it map new memory inside
        # the caller's timed loop)
        NS = 3
        slots = [{k: t.empty(s, dtype=t.float64, device=self.device) for k, (s, _) in
                  shapes.items()} for _ in range(NS)]
        dense_out = [self.alloc(F, dense) for _ in range(2)]  # per compute stream
        labs = [o.labels for o in dense_out] + [
            t.empty((F, nz, ny, nx), dtype=t.uint8, device=self.device)]
        if labels_out is None:
            labels_out = [t.empty((b.n_frames, nz, ny, nx), dtype=t.uint8).pin_memory()
                          for b in batches]
        n_edge = max(1, min(int(edge_pieces), F // 8))  # pieces of >= 8 frames

        def ranges(k):
            n = n_edge if k in (0, nb - 1) else 1
            cut = [F * j // n for j in range(n + 1)]
            return list(zip(cut[:-1], cut[1:]))

        ev_h2d = [[] for _ in range(NS)]       # per input slot: one event per range
        ev_in_free = [None] * NS               # batch done: its input slot may be refilled
        ev_out_free = [None] * NS              # label D2H done: the buffer may be rewritten
        ev_done = {}

        def load(k):
            q = k % NS
            if tuple(host[k]["opacity"].shape) != shapes["opacity"][0]:
                raise ValueError("all batches of a stream must have the same shape")
            with t.cuda.stream(h2d):
                if ev_in_free[q] is not None:
                    h2d.wait_event(ev_in_free[q])
                ev_h2d[q] = []
                for lo, hi in ranges(k):
                    for f, v in host[k].items():
                        slots[q][f][lo:hi].copy_(v[lo:hi], non_blocking=True)
                    ev_h2d[q].append(h2d.record_event())

        part = lambda a, lo, hi: None if a is None else a[lo:hi]
        try:
            load(0)
            for k in range(nb):
                s, q = k & 1, k % NS
                if k + 1 < nb:
                    load(k + 1)
                # n_valid stays on the host: each call copies its range on its own stream
                full = PrimitiveBatch(*(slots[q][f] for f in PrimitiveBatch.FIELDS),
                                      n_valid=batches[k].n_valid)
                out = VoxelizeResult(labs[q], dense_out[s].v_o, dense_out[s].v_c, self.free_code)
                rs = ranges(k)
                used, last_d2h = set(), None
                n_pairs = n_entries = 0
                for j, (lo, hi) in enumerate(rs):
                    # a single range keeps the batch's stream; edge ranges alternate
                    ci = s if len(rs) == 1 else (s + j) & 1
                    comp = comps[ci]
                    with t.cuda.stream(comp):
                        comp.wait_event(ev_h2d[q][j])
                        if ev_out_free[q] is not None:
                            comp.wait_event(ev_out_free[q])
                        if ci != s and ci not in used and k >= 2:
                            comp.wait_event(ev_done[k - 2])  # the dense slot's last user
                        used.add(ci)
                        sub = full if len(rs) == 1 else full.frames(lo, hi)
                        view = out if len(rs) == 1 else VoxelizeResult(
                            out.labels[lo:hi], part(out.v_o, lo, hi), part(out.v_c, lo, hi))
                        r = self(sub, dense=dense, out=view, _slot=ci, _frame0=lo)
                        n_pairs += r.n_pairs
                        n_entries += r.n_entries
                        piece_done = comp.record_event()
                    if k == nb - 1 and len(rs) > 1:  # the last batch's labels per range
                        with t.cuda.stream(d2h):
                            d2h.wait_event(piece_done)
                            labels_out[k][lo:hi].copy_(out.labels[lo:hi], non_blocking=True)
                            last_d2h = d2h.record_event()
                comp = comps[s]
                with t.cuda.stream(comp):
                    for ci in used - {s}:
                        comp.wait_stream(comps[ci])
                    out.n_pairs, out.n_entries = n_pairs, n_entries
                    if on_device is not None:
                        on_device(k, out)
                    done = comp.record_event()
                ev_done[k] = ev_in_free[q] = done
                ev_done.pop(k - 3, None)
                if last_d2h is None:
                    with t.cuda.stream(d2h):
                        d2h.wait_event(done)
                        labels_out[k].copy_(out.labels, non_blocking=True)
                        last_d2h = d2h.record_event()
                ev_out_free[q] = last_d2h
        finally:
            # also on an error: no buffer of this call is released (and
            # reused by the caching allocator) while a copy or compute stream
            # may still use it
            for st in (h2d, d2h, comps[1], comp0):
                st.synchronize()
        comp0.wait_stream(comps[1])
        return labels_out

    # ---- run ----------------------------------------------------------------
    def alloc(self, n_frames: int, dense: bool = True) -> VoxelizeResult:
        t = self.torch
        nx, ny, nz = self.spec.dims
        out = VoxelizeResult(labels=t.empty((n_frames, nz, ny, nx), dtype=t.uint8,
                                            device=self.device), free_code=self.free_code)
        if dense:
            out.v_o = t.empty((n_frames, nz, ny, nx), dtype=t.float32, device=self.device)
            out.v_c = t.empty((n_frames, nz, ny, nx, self.C), dtype=t.float32, device=self.device)
        return out

    def __call__(self, batch: PrimitiveBatch, *, dense: bool = True, bins: bool = False,
                 out: VoxelizeResult | None = None, _slot: int = 0,
                 _frame0: int = 0) -> VoxelizeResult:
        """Voxelize F frames.  Host inputs are copied to the device first
        (non_blocking from pinned memory).  ``out`` may be preallocated with
        ``alloc``; ``dense=False`` keeps v_o/v_c on chip (labels only)."""
        t = self.torch
        if batch.n_classes != self.C:
            raise ValueError(f"batch has {batch.n_classes} classes, voxelizer expects {self.C}")
        with t.cuda.device(self.device):
            try:
                return self._run(batch, dense, bins, out, _slot, _frame0)
            except _lib.SqvError as e:
                # index spaces are 32-bit per call: halve the frames and retry
                if "split frames" not in str(e) or batch.n_frames < 2 or bins:
                    raise
            F, h = batch.n_frames, batch.n_frames // 2
            if out is None:
                out = self.alloc(F, dense)
            part = lambda a, lo, hi: None if a is None else a[lo:hi]
            rs = [self(batch.frames(lo, hi), dense=dense,
                       out=VoxelizeResult(out.labels[lo:hi], part(out.v_o, lo, hi),
                                          part(out.v_c, lo, hi)), _slot=_slot,
                       _frame0=_frame0 + lo)
                  for lo, hi in ((0, h), (h, F))]
            out.free_code = self.free_code
            out.n_pairs = sum(r.n_pairs for r in rs)
            out.n_entries = sum(r.n_entries for r in rs)
            return out

    def _run(self, batch, dense, bins, out, slot=0, frame0=0):
        """One sqv_voxelize call; frame0 = the batch's first frame in the
        caller's batch (a range of it), for error messages."""
        t = self.torch
        db = self.to_device(batch)
        F, N = db.n_frames, db.n_prims
        if out is None:
            out = self.alloc(F, dense)
        out.free_code = self.free_code
        P = _lib.Prims()
        P.mu, P.scale, P.rot = db.mu.data_ptr(), db.scale.data_ptr(), db.rot.data_ptr()
        P.opacity, P.eps, P.logits = db.opacity.data_ptr(), db.eps.data_ptr(), db.logits.data_ptr()
        P.n_valid = None if db.n_valid is None else db.n_valid.data_ptr()
        P.n_frames, P.n_prims, P.n_classes = F, N, self.C
        O = _lib.Outputs()
        O.labels = out.labels.data_ptr()
        O.v_o = out.v_o.data_ptr() if out.v_o is not None else None
        O.v_c = out.v_c.data_ptr() if out.v_c is not None else None
        B = _lib.Bins()
        bins_t = None
        if bins:
            T = self.tiles_per_frame
            bins_t = {"windows": t.empty((F, N, 6), dtype=t.int32, device=self.device),
                      "tile_off": t.empty(F * T + 1, dtype=t.int32, device=self.device),
                      "prim_ids": t.empty(1, dtype=t.int32, device=self.device)}
            B.windows = bins_t["windows"].data_ptr()
            B.tile_off = bins_t["tile_off"].data_ptr()
        stream = _lib.stream_ptr(self.device)
        need = ctypes.c_size_t(0)
        bad_prim = ctypes.c_int64(-1)
        bad_bits = ctypes.c_int32(0)
        ws_bytes = int(self.L.sqv_workspace_bytes(F, N, self.C, ctypes.byref(self._grid), 0))
        for _attempt in range(4):
            ws = self._workspace(ws_bytes, slot)
            if bins:
                B.prim_ids = bins_t["prim_ids"].data_ptr()
                B.capacity = bins_t["prim_ids"].numel()
            rc = self.L.sqv_voxelize(ctypes.byref(P), ctypes.byref(self._grid),
                                     ctypes.byref(self._cfg), ctypes.byref(O), ctypes.byref(B),
                                     ws.data_ptr(), ws.numel(), ctypes.byref(need),
                                     ctypes.byref(bad_prim), ctypes.byref(bad_bits), stream)
            if rc == _lib.SQV_ERR_WORKSPACE:
                ws_bytes = int(need.value)
                continue
            if rc == _lib.SQV_ERR_CAPACITY and bins:
                bins_t["prim_ids"] = t.empty(max(1, int(B.n_entries)), dtype=t.int32,
                                             device=self.device)
                continue
            if rc == _lib.SQV_ERR_INVALID_PRIM:
                f, i = divmod(int(bad_prim.value), max(N, 1))
                f += frame0
                raise ValueError(f"frame {f} primitive {i}: "
                                 f"{bad_bits_message(int(bad_bits.value))}")
            _lib.check(rc, "sqv_voxelize")
            break
        else:
            raise RuntimeError("sqv_voxelize: workspace negotiation did not converge")
        out.n_pairs, out.n_entries = int(B.n_pairs), int(B.n_entries)
        if bins:
            bins_t["prim_ids"] = bins_t["prim_ids"][: out.n_entries]
            out.bins = bins_t
        return out


# ---- conversions to the SPEC's host types ---------------------------------

def _logical(a: np.ndarray) -> np.ndarray:
    """(nz, ny, nx[, C]) x-fastest memory -> (nx, ny, nz[, C]) view."""
    return a.transpose(2, 1, 0, 3) if a.ndim == 4 else a.transpose(2, 1, 0)


def labels_to_host(labels_u8: np.ndarray, free_code: int, free_index: int) -> np.ndarray:
    if free_code == free_index:
        return labels_u8
    out = labels_u8.astype(np.int64)
    out[labels_u8 == free_code] = free_index
    return out


def _as_batch(scene) -> tuple[PrimitiveBatch, ClassTable]:
    if isinstance(scene, PrimitiveBatch):
        return scene, ClassTable.numbered(scene.n_classes)
    if hasattr(scene, "primitives") and hasattr(scene, "classes"):
        return PrimitiveBatch.from_scene(scene), scene.classes
    raise TypeError("scene must be a Scene (sqocc.core or ours) or a PrimitiveBatch")


def _run_scene(scene, spec, cfg, truncate):
    batch, classes = _as_batch(scene)
    if batch.n_frames != 1:
        raise ValueError("voxelize() takes one scene; use Voxelizer for batches")
    vox = Voxelizer(spec, cfg, len(classes), classes.free_index, truncate=truncate)
    r = vox(batch, dense=True)
    lab = r.labels[0].cpu().numpy()
    v_o = r.v_o[0].cpu().numpy()
    v_c = r.v_c[0].cpu().numpy()
    lab = labels_to_host(lab, r.free_code, classes.free_index)
    return (SemanticGrid(_logical(lab), spec, classes),
            DenseGrids(_logical(v_o), _logical(v_c), spec))


def voxelize(scene, spec: VoxelGridSpec = VoxelGridSpec(),
             cfg: VoxelizeConfig = VoxelizeConfig()) -> tuple[SemanticGrid, DenseGrids]:
    """Eqs. 8-9 with the truncated window, then finalize."""
    return _run_scene(scene, spec, cfg, truncate=True)


def voxelize_bruteforce(scene, spec: VoxelGridSpec = VoxelGridSpec(),
                        cfg: VoxelizeConfig = VoxelizeConfig()) -> tuple[SemanticGrid, DenseGrids]:
    """Untruncated gather: every primitive over the whole
    grid, same sigma = 0 skip and finalize as voxelize."""
    return _run_scene(scene, spec, cfg, truncate=False)


def finalize(dense: DenseGrids, tau: float, classes: ClassTable,
             spec: VoxelGridSpec | None = None) -> SemanticGrid:
    """Labels from dense grids — the device finalize kernel.

    The SemanticGrid's geometry (it feeds ray_iou and the SQOC header) is
    ``spec``, else ``dense.spec`` (set by voxelize), else the Occ3D default
    when the dims match it; any other grid needs one of the two, and
    finalize raises rather than attach the default origin/resolution to it."""
    import torch
    dev = _lib.require_cuda()
    L = _lib.lib()
    if not (float(tau) >= 0.0):
        raise ValueError("tau must be >= 0")
    C = len(classes)
    v_o = np.asarray(dense.v_o)
    v_c = np.asarray(dense.v_c)
    if v_c.shape[:-1] != v_o.shape or v_c.shape[-1] != C:
        raise ValueError("dense grids and classes are inconsistent")
    shape = v_o.shape
    # memory order of the logical (nx, ny, nz) view: x-fastest -> C order of (nz, ny, nx)
    vo_mem = np.ascontiguousarray(v_o.transpose(2, 1, 0), np.float32)
    vc_mem = np.ascontiguousarray(v_c.transpose(2, 1, 0, 3), np.float32)
    t_vo = torch.from_numpy(vo_mem).to(dev)
    t_vc = torch.from_numpy(vc_mem).to(dev)
    code = free_code_for(classes.free_index, C)
    lab = torch.empty(vo_mem.shape, dtype=torch.uint8, device=dev)
    _lib.check(L.sqv_finalize(t_vo.data_ptr(), t_vc.data_ptr(), vo_mem.size, C, float(tau), code,
                              lab.data_ptr(), _lib.stream_ptr(dev)), "sqv_finalize")
    lab_h = labels_to_host(lab.cpu().numpy(), code, classes.free_index)
    return SemanticGrid(_logical(lab_h), _grid_spec_for(shape, spec, dense), classes)


def _grid_spec_for(shape, spec, dense) -> VoxelGridSpec:
    spec = spec if spec is not None else getattr(dense, "spec", None)
    if spec is None:
        if tuple(shape) != VoxelGridSpec().dims:
            raise ValueError(f"dense grids of dims {tuple(shape)} carry no grid geometry: "
                             "pass spec= (the default Occ3D origin/resolution only "
                             "applies to 200x200x16)")
        return VoxelGridSpec()
    if tuple(spec.dims) != tuple(shape):
        raise ValueError(f"spec dims {spec.dims} differ from the dense grids' {tuple(shape)}")
    return spec


def truncation_report(batch: PrimitiveBatch, spec: VoxelGridSpec = VoxelGridSpec(),
                      cfg: VoxelizeConfig = VoxelizeConfig()) -> dict:
    """Truncated voxelize vs voxelize_bruteforce on the device (SPEC.md:376,
    cmd_voxelize --oracle).

    Returns the max |dv_o| (omitted mass), the label mismatch rate, whether
    every mismatching voxel lost positive mass (truncation soundness), and a
    per-primitive tail bound: outside its window a primitive's local scaled
    coordinates satisfy |x'|_inf >= (r - 1/2) res / (sqrt(3) max(s)), so
    sigma * exp(-F) <= sigma * exp(-((r - 1/2) res / (sqrt(3) max(s)))^(2/eps1)).
    """
    import torch
    C = batch.n_classes
    tr = Voxelizer(spec, cfg, C, truncate=True)(batch)
    bf = Voxelizer(spec, cfg, C, truncate=False)(batch)
    dvo = (bf.v_o.double() - tr.v_o.double())
    diff = tr.labels != bf.labels
    sound = bool(torch.all(dvo[diff] > 0).item()) if bool(diff.any()) else True
    sc = np.asarray(batch.scale, np.float64)
    e1 = np.clip(np.asarray(batch.eps, np.float64)[..., 0], 0.2, 2.0)
    smax = sc.max(-1)
    r = cfg.neighborhood_radius + np.ceil(smax * cfg.window_extent / spec.resolution)
    reach = np.maximum(r - 0.5, 0.0) * spec.resolution / (np.sqrt(3.0) * smax)
    tail = np.asarray(batch.opacity, np.float64) * np.exp(-np.power(reach, 2.0 / e1))
    if batch.n_valid is not None:
        nv = np.asarray(batch.n_valid)
        tail = np.where(np.arange(tail.shape[1])[None, :] < nv[:, None], tail, 0.0)
    return {"max_omitted_mass": float(dvo.max().item()),
            "min_dvo": float(dvo.min().item()),
            "label_mismatch_rate": float(diff.double().mean().item()),
            "sound": sound,
            "max_single_primitive_tail_bound": float(tail.max()),
            "sum_tail_bound": float(tail.sum(-1).max())}
