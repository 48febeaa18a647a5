"""ctypes binding of libsqv.so (include/sqv.h).

The product path has no CPU fallback: if the library is missing or no CUDA
device is present, every entry point raises.  torch is used only for device
memory and the current stream (plumbing); the compute is libsqv's kernels.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# SQV_LIB: an alternative build of the same library (A/B runs of compile-time
# variants, scripts/gpu_ab_env.sh); the default is the in-tree build
LIB_PATH = os.environ.get("SQV_LIB") or os.path.join(_HERE, "_build", "libsqv.so")

SQV_OK = 0
SQV_ERR_ARG = -1
SQV_ERR_CUDA = -2
SQV_ERR_WORKSPACE = -3
SQV_ERR_INVALID_PRIM = -4
SQV_ERR_UNSUPPORTED = -5
SQV_ERR_CAPACITY = -6
TILE = (8, 8, 16)
MAX_CLASSES = 32

_c_p = ctypes.c_void_p
_i32, _i64, _f64 = ctypes.c_int32, ctypes.c_int64, ctypes.c_double


class Grid(ctypes.Structure):
    _fields_ = [("origin", _f64 * 3), ("dims", _i32 * 3), ("resolution", _f64)]


class Cfg(ctypes.Structure):
    _fields_ = [("tau", _f64), ("neighborhood_radius", _i32), ("truncate", _i32),
                ("semantic_mode", _i32), ("free_label", _i32), ("window_extent", _f64),
                ("precision", _i32)]


class Prims(ctypes.Structure):
    _fields_ = [("mu", _c_p), ("scale", _c_p), ("rot", _c_p), ("opacity", _c_p), ("eps", _c_p),
                ("logits", _c_p), ("n_valid", _c_p), ("n_frames", _i32), ("n_prims", _i32),
                ("n_classes", _i32)]


class Outputs(ctypes.Structure):
    _fields_ = [("labels", _c_p), ("v_o", _c_p), ("v_c", _c_p)]


class Bins(ctypes.Structure):
    _fields_ = [("windows", _c_p), ("tile_off", _c_p), ("prim_ids", _c_p), ("capacity", _i64),
                ("n_entries", _i64), ("n_pairs", _i64)]


class SqvError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"libsqv error {code}: {msg}")
        self.code = code


class RayHits(ctypes.Structure):
    _fields_ = [("d_pred", _c_p), ("c_pred", _c_p), ("d_gt", _c_p), ("c_gt", _c_p)]


_lib = None


def lib():
    """Load libsqv.so (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"{LIB_PATH} is missing: build it with `python -m paper_2511_17361_b200.build` "
            "(or __graft_entry__.build()).  There is no CPU fallback.")
    L = ctypes.CDLL(LIB_PATH)
    L.sqv_abi_version.restype = ctypes.c_int
    L.sqv_last_error.restype = ctypes.c_char_p
    L.sqv_launch_count.restype = _i64
    L.sqv_tiles_per_frame.argtypes = [ctypes.POINTER(Grid)]
    L.sqv_tiles_per_frame.restype = _i64
    L.sqv_workspace_bytes.argtypes = [_i32, _i32, _i32, ctypes.POINTER(Grid), _i64]
    L.sqv_workspace_bytes.restype = ctypes.c_size_t
    L.sqv_voxelize.argtypes = [ctypes.POINTER(Prims), ctypes.POINTER(Grid), ctypes.POINTER(Cfg),
                               ctypes.POINTER(Outputs), ctypes.POINTER(Bins), _c_p,
                               ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t),
                               ctypes.POINTER(_i64), ctypes.POINTER(_i32), _c_p]
    L.sqv_finalize.argtypes = [_c_p, _c_p, _i64, _i32, _f64, _i32, _c_p, _c_p]
    L.sqv_confusion.argtypes = [_c_p, _c_p, _i64, _i32, _i32, _c_p, _c_p]
    L.sqv_density.argtypes = [ctypes.POINTER(Prims), _c_p, _c_p, _i64, _c_p, _c_p, _c_p]
    L.sqv_profile_enable.argtypes = [ctypes.c_int]
    L.sqv_profile_read.argtypes = [_c_p, ctypes.POINTER(_i64), ctypes.c_int]
    L.sqv_microbench.argtypes = [ctypes.c_int, ctypes.POINTER(_f64), _c_p]
    L.sqv_stats_attach.argtypes = [_c_p]
    L.sqv_ray_iou.argtypes = [_c_p, _c_p, _i32, ctypes.POINTER(Grid), _i32, _c_p, _c_p, _i64,
                              _c_p, _i32, _c_p, ctypes.POINTER(RayHits), _c_p]
    L.sqv_gen_frames.argtypes = [ctypes.c_uint64, _i64, _i32, _i32, _i32, ctypes.POINTER(Grid),
                                 _f64, _f64, _f64, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p]
    for f in ("sqv_voxelize", "sqv_finalize", "sqv_confusion", "sqv_density",
              "sqv_profile_enable", "sqv_profile_read", "sqv_microbench", "sqv_ray_iou",
              "sqv_gen_frames", "sqv_stats_attach"):
        getattr(L, f).restype = ctypes.c_int
    if L.sqv_abi_version() != 1:
        raise RuntimeError("libsqv ABI version mismatch")
    _lib = L
    return L


EXPORTED = ("sqv_abi_version", "sqv_last_error", "sqv_launch_count", "sqv_tiles_per_frame",
            "sqv_workspace_bytes", "sqv_voxelize", "sqv_finalize", "sqv_confusion",
            "sqv_density", "sqv_profile_enable", "sqv_profile_read", "sqv_microbench",
            "sqv_ray_iou", "sqv_gen_frames", "sqv_stats_attach")


def last_error() -> str:
    return lib().sqv_last_error().decode(errors="replace")


def check(rc: int, what: str = "") -> None:
    if rc != SQV_OK:
        raise SqvError(rc, f"{what}: {last_error()}" if what else last_error())


def launch_count() -> int:
    return int(lib().sqv_launch_count())


def require_cuda(device=None):
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2511_17361_b200 needs a CUDA device (B200); there is no CPU "
                           "fallback")
    return torch.device(device) if device is not None else torch.device("cuda",
                                                                        torch.cuda.current_device())


def stream_ptr(device=None) -> int:
    import torch
    return torch.cuda.current_stream(device).cuda_stream


def profile_enable(on: bool = True) -> None:
    check(lib().sqv_profile_enable(int(on)), "sqv_profile_enable")


def profile_read(reset: bool = False) -> dict:
    """Accumulated stage device times (ms) of sqv_voxelize calls since the last reset."""
    import numpy as np
    ms = np.zeros(5, np.float64)
    calls = _i64(0)
    check(lib().sqv_profile_read(ms.ctypes.data_as(_c_p), ctypes.byref(calls), int(reset)),
          "sqv_profile_read")
    return {"prep_scan_ms": ms[0], "bin_sort_ms": ms[1], "eval_ms": ms[2], "total_ms": ms[3],
            "eval_kernel_ms": ms[4], "calls": int(calls.value)}


def microbench(which: int) -> float:
    """Measured pipe rate on the current GPU: 0 -> MUFU ops/s, 1 -> FFMA lanes/s."""
    v = _f64(0.0)
    check(lib().sqv_microbench(int(which), ctypes.byref(v), stream_ptr()), "sqv_microbench")
    return float(v.value)


def stats_attach(counters) -> None:
    """Attach an int64[2] device tensor as the evaluator work counters
    (include/sqv.h sqv_stats_attach); None detaches."""
    check(lib().sqv_stats_attach(None if counters is None else counters.data_ptr()),
          "sqv_stats_attach")
