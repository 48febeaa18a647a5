"""Domain types of the voxelization path, structure-of-arrays first.

Mirrors the reference's primitive types so existing callers keep working:

- ``SuperQuadric``  — /root/reference/pkg/src/sqocc/core.py:119-185
- ``ClassTable``    — core.py:188-212
- ``Scene``         — core.py:215-230
- ``EPS_MIN/EPS_MAX/F_CAP`` — core.py:16-23

Same fields, same validation order and the same ``ValueError`` messages.  The
difference is the representation the device consumes: ``PrimitiveBatch`` holds
F frames x N primitives as FP64 arrays (the layout of ``sqv_prims`` in
include/sqv.h) and validates them vectorially, so a 2,000-primitive frame is
packed without constructing 2,000 Python objects (the reference spends
~76 us per ``SuperQuadric``).

Inputs that come straight from SoA arrays (``PrimitiveBatch``) are validated
on the device by the prep kernel and reported with the messages below.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Iterable, Sequence

import numpy as np

EPS_MIN = 0.2   # core.py:18
EPS_MAX = 2.0   # core.py:19
F_CAP = 1e30    # core.py:23

# Validation failure bits reported by the device prep kernel (include/sqv.h
# SQV_BAD_*), in the order SuperQuadric.__post_init__ checks them
# (core.py:147-159, quat_normalize core.py:33-34).
BAD_BITS_MESSAGES = (
    (1, "mu/scale must be finite"),
    (2, "scale components must be strictly positive"),
    (4, "logits must be finite"),
    (8, "opacity must lie in [0, 1]"),
    (16, "cannot normalize near-zero quaternion"),
    (32, "eps1/eps2 must be finite"),
)


def bad_bits_message(bits: int) -> str:
    for bit, msg in BAD_BITS_MESSAGES:
        if bits & bit:
            return msg
    return "invalid primitive"


def _quat_normalize(q: np.ndarray) -> np.ndarray:
    q = np.asarray(q, dtype=np.float64)
    n = np.sqrt(np.sum(q * q, axis=-1, keepdims=True))
    if np.any(n < 1e-12):
        raise ValueError("cannot normalize near-zero quaternion")
    return q / n


def _frozen(a) -> np.ndarray:
    a = np.array(a, dtype=np.float64)
    a.flags.writeable = False
    return a


@dataclass(frozen=True)
class SuperQuadric:
    """One primitive (core.py:119-185): mu, scale, rot (w,x,y,z, local-to-world),
    opacity in [0,1], logits (C,), eps1/eps2 clamped to [EPS_MIN, EPS_MAX]."""

    mu: np.ndarray
    scale: np.ndarray
    rot: np.ndarray
    opacity: float
    logits: np.ndarray
    eps1: float
    eps2: float
    eps_clamped: bool = field(init=False, default=False)

    def __post_init__(self):
        mu, scale, logits = _frozen(self.mu), _frozen(self.scale), _frozen(self.logits)
        if mu.shape != (3,) or scale.shape != (3,):
            raise ValueError("mu and scale must be 3-vectors")
        if logits.ndim != 1:
            raise ValueError("logits must be a 1-D class-score vector")
        if not (np.isfinite(mu).all() and np.isfinite(scale).all()):
            raise ValueError("mu/scale must be finite")
        if not (scale > 0.0).all():
            raise ValueError("scale components must be strictly positive")
        if not np.isfinite(logits).all():
            raise ValueError("logits must be finite")
        opacity = float(self.opacity)
        if not (0.0 <= opacity <= 1.0):
            raise ValueError("opacity must lie in [0, 1]")
        rot = _quat_normalize(self.rot)
        rot.flags.writeable = False
        e1, e2 = float(self.eps1), float(self.eps2)
        clamped = not (EPS_MIN <= e1 <= EPS_MAX and EPS_MIN <= e2 <= EPS_MAX)
        set_ = object.__setattr__
        set_(self, "mu", mu)
        set_(self, "scale", scale)
        set_(self, "rot", rot)
        set_(self, "opacity", opacity)
        set_(self, "logits", logits)
        set_(self, "eps1", min(max(e1, EPS_MIN), EPS_MAX))
        set_(self, "eps2", min(max(e2, EPS_MIN), EPS_MAX))
        set_(self, "eps_clamped", clamped)

    @property
    def num_classes(self) -> int:
        return self.logits.shape[0]

    def rotation_matrix(self) -> np.ndarray:
        return quat_to_matrix(self.rot)

    def world_to_local_matrix(self) -> np.ndarray:
        return quat_to_matrix(self.rot).T


@dataclass(frozen=True)
class ClassTable:
    """Class names + free sentinel outside [0, C), default C (core.py:188-212)."""

    names: tuple
    free_index: int | None = None

    def __post_init__(self):
        names = tuple(str(n) for n in self.names)
        if len(names) < 1:
            raise ValueError("need at least one class")
        if len(set(names)) != len(names):
            raise ValueError("class names must be unique")
        free = len(names) if self.free_index is None else int(self.free_index)
        if 0 <= free < len(names):
            raise ValueError("free_index must lie outside [0, C)")
        object.__setattr__(self, "names", names)
        object.__setattr__(self, "free_index", free)

    def __len__(self) -> int:
        return len(self.names)

    @staticmethod
    def numbered(C: int) -> "ClassTable":
        return ClassTable(tuple(f"class_{k}" for k in range(C)))


@dataclass
class Scene:
    """Primitives over a shared class table (core.py:215-230)."""

    primitives: list
    classes: ClassTable

    def __post_init__(self):
        C = len(self.classes)
        for i, sq in enumerate(self.primitives):
            if sq.num_classes != C:
                raise ValueError(f"primitive {i} has {sq.num_classes} logits, expected {C}")

    def __len__(self) -> int:
        return len(self.primitives)


def quat_to_matrix(q) -> np.ndarray:
    """Local-to-world rotation of unit quaternion(s) (w,x,y,z), core.py:55-65.
    Vectorised over leading axes."""
    q = np.asarray(q, dtype=np.float64)
    w, x, y, z = q[..., 0], q[..., 1], q[..., 2], q[..., 3]
    R = np.empty(q.shape[:-1] + (3, 3))
    R[..., 0, 0] = 1.0 - 2.0 * (y * y + z * z)
    R[..., 0, 1] = 2.0 * (x * y - w * z)
    R[..., 0, 2] = 2.0 * (x * z + w * y)
    R[..., 1, 0] = 2.0 * (x * y + w * z)
    R[..., 1, 1] = 1.0 - 2.0 * (x * x + z * z)
    R[..., 1, 2] = 2.0 * (y * z - w * x)
    R[..., 2, 0] = 2.0 * (x * z - w * y)
    R[..., 2, 1] = 2.0 * (y * z + w * x)
    R[..., 2, 2] = 1.0 - 2.0 * (x * x + y * y)
    return R


class PrimitiveBatch:
    """F frames x N primitives as FP64 structure-of-arrays (sqv_prims layout).

    mu [F,N,3], scale [F,N,3], rot [F,N,4] (w,x,y,z; need not be normalised),
    opacity [F,N], eps [F,N,2] (eps1, eps2; clamped on the device),
    logits [F,N,C], n_valid [F] int32 or None (ragged frames: primitives
    i >= n_valid[f] are ignored).

    Arrays may be NumPy arrays or torch tensors (host or CUDA); the voxelizer
    moves host arrays to the device itself.
    """

    FIELDS = ("mu", "scale", "rot", "opacity", "eps", "logits")

    def __init__(self, mu, scale, rot, opacity, eps, logits, n_valid=None):
        self.mu, self.scale, self.rot = mu, scale, rot
        self.opacity, self.eps, self.logits = opacity, eps, logits
        self.n_valid = n_valid
        F, N = tuple(opacity.shape)
        C = logits.shape[-1]
        shapes = {"mu": (F, N, 3), "scale": (F, N, 3), "rot": (F, N, 4), "opacity": (F, N),
                  "eps": (F, N, 2), "logits": (F, N, C)}
        for k, s in shapes.items():
            if tuple(getattr(self, k).shape) != s:
                raise ValueError(f"{k} must have shape {s}, got {tuple(getattr(self, k).shape)}")
        if C < 1:
            raise ValueError("need at least one class")
        if n_valid is not None and tuple(n_valid.shape) != (F,):
            raise ValueError(f"n_valid must have shape ({F},)")

    @property
    def n_frames(self) -> int:
        return int(self.opacity.shape[0])

    @property
    def n_prims(self) -> int:
        return int(self.opacity.shape[1])

    @property
    def n_classes(self) -> int:
        return int(self.logits.shape[-1])

    def frames(self, start: int, stop: int) -> "PrimitiveBatch":
        nv = None if self.n_valid is None else self.n_valid[start:stop]
        return PrimitiveBatch(*(getattr(self, k)[start:stop] for k in self.FIELDS), n_valid=nv)

    # ---- construction from the reference's object model ----------------
    @staticmethod
    def from_scene(scene) -> "PrimitiveBatch":
        """Pack a Scene (ours or the reference's sqocc.core.Scene) as one frame."""
        return PrimitiveBatch.from_scenes([scene])

    @staticmethod
    def from_scenes(scenes: Sequence) -> "PrimitiveBatch":
        """Pack several scenes (same class count) as frames; ragged -> n_valid."""
        if len(scenes) == 0:
            raise ValueError("need at least one scene")
        C = len(scenes[0].classes)
        for s in scenes:
            if len(s.classes) != C:
                raise ValueError("all scenes must share the class count")
        F = len(scenes)
        N = max(1, max(len(s.primitives) for s in scenes))
        mu = np.zeros((F, N, 3))
        scale = np.ones((F, N, 3))
        rot = np.zeros((F, N, 4))
        rot[..., 0] = 1.0
        opacity = np.zeros((F, N))
        eps = np.ones((F, N, 2))
        logits = np.zeros((F, N, C))
        n_valid = np.zeros(F, np.int32)
        for f, s in enumerate(scenes):
            prims = s.primitives
            n = len(prims)
            n_valid[f] = n
            if n == 0:
                continue
            mu[f, :n] = [p.mu for p in prims]
            scale[f, :n] = [p.scale for p in prims]
            rot[f, :n] = [p.rot for p in prims]
            opacity[f, :n] = [p.opacity for p in prims]
            eps[f, :n, 0] = [p.eps1 for p in prims]
            eps[f, :n, 1] = [p.eps2 for p in prims]
            logits[f, :n] = [p.logits for p in prims]
        ragged = not np.all(n_valid == N)
        return PrimitiveBatch(mu, scale, rot, opacity, eps, logits,
                              n_valid=n_valid if ragged else None)

    @staticmethod
    def from_primitives(prims: Iterable, n_classes: int | None = None) -> "PrimitiveBatch":
        prims = list(prims)
        C = n_classes if n_classes is not None else (prims[0].num_classes if prims else 1)
        return PrimitiveBatch.from_scenes([Scene(prims, ClassTable.numbered(C))])

    # ---- host-side validation (vectorised; device prep re-checks) -------
    def validate(self) -> None:
        """Raise ValueError with the reference's message for the first invalid
        primitive (core.py:147-159 order).  NumPy inputs only."""
        bits = validation_bits(self)
        bad = np.flatnonzero(bits)
        if bad.size:
            i = int(bad[0])
            f, n = divmod(i, self.n_prims)
            raise ValueError(f"frame {f} primitive {n}: {bad_bits_message(int(bits.flat[i]))}")


def validation_bits(b: PrimitiveBatch) -> np.ndarray:
    """Per-primitive failure bits [F,N] (include/sqv.h SQV_BAD_*), NumPy."""
    mu, scale, rot = (np.asarray(getattr(b, k), np.float64) for k in ("mu", "scale", "rot"))
    opacity, eps, logits = (np.asarray(getattr(b, k), np.float64)
                            for k in ("opacity", "eps", "logits"))
    bits = np.zeros(opacity.shape, np.int32)
    fin = np.isfinite(mu).all(-1) & np.isfinite(scale).all(-1)
    bits |= np.where(~fin, 1, 0).astype(np.int32)
    bits |= np.where(fin & ~(scale > 0).all(-1), 2, 0).astype(np.int32)
    bits |= np.where(~np.isfinite(logits).all(-1), 4, 0).astype(np.int32)
    bits |= np.where(~((opacity >= 0) & (opacity <= 1)), 8, 0).astype(np.int32)
    qn = np.sqrt(np.sum(rot * rot, axis=-1))
    bits |= np.where(~(qn >= 1e-12), 16, 0).astype(np.int32)
    bits |= np.where(~np.isfinite(eps).all(-1), 32, 0).astype(np.int32)
    if b.n_valid is not None:
        nv = np.asarray(b.n_valid)
        idx = np.arange(bits.shape[1])[None, :]
        bits[idx >= nv[:, None]] = 0
    return bits
