"""Diagnostics: the previous Voxelizer.stream (double-buffered, no edge ranges)
as a free function, for A/B timing against the current one."""
import numpy as np
from paper_2511_17361_b200.core import PrimitiveBatch
from paper_2511_17361_b200.voxelize import VoxelizeResult


def stream(self, batches, *, dense: bool = True, on_device=None, labels_out=None):
    """Voxelize a sequence of host batches (pinned torch tensors for real
    overlap) with copies overlapped: the H2D copy of batch k+1 and the D2H
    copy of batch k-1's labels run on two copy streams while batch k is
    evaluated; consecutive batches alternate two compute streams (the
    current one and a side stream, as in ``run_many``) so a batch's
    binning overlaps the previous evaluation.  ``on_device(k, result)`` is
    called on batch k's compute stream right after it (e.g. confusion
    counts).
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
    slots = [{k: t.empty(s, dtype=t.float64, device=self.device) for k, (s, _) in
              shapes.items()} for _ in range(2)]
    outs = [self.alloc(batches[0].n_frames, dense) for _ in range(2)]
    if labels_out is None:
        labels_out = [t.empty((b.n_frames, nz, ny, nx), dtype=t.uint8).pin_memory()
                      for b in batches]
    ev_h2d = [None, None]
    ev_in_free = [None, None]
    ev_out_free = [None, None]

    def load(k):
        s = k & 1
        if tuple(host[k]["opacity"].shape) != shapes["opacity"][0]:
            raise ValueError("all batches of a stream must have the same shape")
        with t.cuda.stream(h2d):
            if ev_in_free[s] is not None:
                h2d.wait_event(ev_in_free[s])
            for f, v in host[k].items():
                slots[s][f].copy_(v, non_blocking=True)
            ev_h2d[s] = h2d.record_event()

    load(0)
    for k in range(nb):
        s = k & 1
        if k + 1 < nb:
            load(k + 1)
        comp = comps[s]
        with t.cuda.stream(comp):
            comp.wait_event(ev_h2d[s])
            if ev_out_free[s] is not None:
                comp.wait_event(ev_out_free[s])
            nv = batches[k].n_valid
            db = PrimitiveBatch(*(slots[s][f] for f in PrimitiveBatch.FIELDS),
                                n_valid=None if nv is None else self._dev(nv, t.int32))
            res = self(db, dense=dense, out=outs[s], _slot=s)
            if on_device is not None:
                on_device(k, res)
            done = comp.record_event()
        ev_in_free[s] = done
        with t.cuda.stream(d2h):
            d2h.wait_event(done)
            labels_out[k].copy_(outs[s].labels, non_blocking=True)
            ev_out_free[s] = d2h.record_event()
    d2h.synchronize()
    comps[1].synchronize()
    comp0.wait_stream(comps[1])
    comp0.synchronize()
    return labels_out

