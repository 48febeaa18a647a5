"""SceneFile JSON-lines: the input format of cmd_voxelize.

Line 1 (header):  {"version": 1, "classes": ["name", ...]}
Then one record per primitive:
    {"mu": [3], "scale": [3], "quat": [4 w,x,y,z], "opacity": s,
     "eps": [eps1, eps2], "logits": [C]}

``read`` parses straight into a one-frame ``PrimitiveBatch`` (no per-object
SuperQuadric construction), rejects NaN/Inf and reports
malformed records with their line number.  ``write`` is atomic and
deterministic (floats written with repr, which round-trips exactly).
"""
from __future__ import annotations

import json
import math
import os
import tempfile

import numpy as np

from .core import ClassTable, PrimitiveBatch

VERSION = 1


def _reject_constant(name):
    raise ValueError(f"non-finite number {name} is not allowed")


def read(path: str) -> tuple[PrimitiveBatch, ClassTable]:
    mu, scale, quat, opacity, eps, logits = [], [], [], [], [], []
    with open(path) as fh:
        lines = fh.read().splitlines()
    if not lines:
        raise ValueError(f"{path}:1: missing header")
    try:
        hdr = json.loads(lines[0], parse_constant=_reject_constant)
        classes = ClassTable(tuple(hdr["classes"]))
        if int(hdr.get("version", VERSION)) != VERSION:
            raise ValueError("unsupported SceneFile version")
    except (KeyError, TypeError, ValueError) as e:
        raise ValueError(f"{path}:1: bad header: {e}") from None
    C = len(classes)
    for ln, line in enumerate(lines[1:], start=2):
        if not line.strip():
            continue
        try:
            r = json.loads(line, parse_constant=_reject_constant)
            m, s, q = (np.asarray(r[k], np.float64) for k in ("mu", "scale", "quat"))
            e, lg = np.asarray(r["eps"], np.float64), np.asarray(r["logits"], np.float64)
            o = float(r["opacity"])
            if m.shape != (3,) or s.shape != (3,) or q.shape != (4,) or e.shape != (2,):
                raise ValueError("field shapes")
            if lg.shape != (C,):
                raise ValueError(f"{lg.size} logits, expected {C}")
            vals = np.concatenate([m, s, q, e, lg, [o]])
            if not np.all(np.isfinite(vals)):
                raise ValueError("non-finite value")
        except (KeyError, TypeError, ValueError) as ex:
            raise ValueError(f"{path}:{ln}: malformed record: {ex}") from None
        mu.append(m), scale.append(s), quat.append(q), opacity.append(o), eps.append(e)
        logits.append(lg)
    n = len(mu)
    if n == 0:  # header only: an empty scene (SPEC.md:597 n=0)
        b = PrimitiveBatch(np.zeros((1, 1, 3)), np.ones((1, 1, 3)),
                           np.array([[[1.0, 0, 0, 0]]]), np.zeros((1, 1)), np.ones((1, 1, 2)),
                           np.zeros((1, 1, C)), n_valid=np.zeros(1, np.int32))
        return b, classes
    f = lambda a: np.asarray(a, np.float64)[None]
    return PrimitiveBatch(f(mu), f(scale), f(quat), f(opacity), f(eps), f(logits)), classes


def write(path: str, batch: PrimitiveBatch, classes: ClassTable, frame: int = 0) -> None:
    n = batch.n_prims if batch.n_valid is None else int(np.asarray(batch.n_valid)[frame])
    g = {k: np.asarray(getattr(batch, k))[frame] for k in PrimitiveBatch.FIELDS}
    out = [json.dumps({"version": VERSION, "classes": list(classes.names)})]
    for i in range(n):
        rec = {"mu": [float(v) for v in g["mu"][i]], "scale": [float(v) for v in g["scale"][i]],
               "quat": [float(v) for v in g["rot"][i]], "opacity": float(g["opacity"][i]),
               "eps": [float(v) for v in g["eps"][i]],
               "logits": [float(v) for v in g["logits"][i]]}
        out.append(json.dumps(rec))
    d = os.path.dirname(os.path.abspath(path))
    fd, tmp = tempfile.mkstemp(dir=d, prefix=".scene.")
    try:
        with os.fdopen(fd, "w") as fh:
            fh.write("\n".join(out) + "\n")
        os.replace(tmp, path)
    except BaseException:
        if os.path.exists(tmp):
            os.unlink(tmp)
        raise
