"""The ``sqocc`` command line of SPEC.md:550-619 (cli-io) for the commands
on the voxelization path: the callers and file formats either side of it.

    python -m paper_2511_17361_b200 gen-scene --seed 7 --n 1600 --out scene.jsonl
    python -m paper_2511_17361_b200 voxelize --scene scene.jsonl --out grid.sqoc [--oracle]
    python -m paper_2511_17361_b200 metrics --pred a.sqoc --gt b.sqoc [--thresholds 1,2,4]
    python -m paper_2511_17361_b200 bench --scene scene.jsonl [--repetitions 20]

* ``gen-scene`` — ``gen_scene(seed, n, grid spec)`` written
  as a SceneFile; same seed -> byte-identical file.
* ``voxelize`` — ``cmd_voxelize``: SceneFile -> voxelize
  on the B200 -> SQOC grid, plus timing; ``--oracle`` also
  runs ``voxelize_bruteforce`` and reports max |dv_o| vs the truncated path.
* ``metrics`` — ``cmd_metrics``: IoU, per-class IoU, mIoU
  (confusion counts on the device) and RayIoU of two SQOC grids.
* ``bench`` — ``cmd_bench``: wall-time percentiles of
  voxelize on one scene and the speed-up over the untruncated bruteforce.

Flags keep the SPEC spellings: ``--scene --out --grid-origin x,y,z
--grid-dims nx,ny,nz --resolution --tau --neighborhood --thresholds csv
--seed --oracle --format json|text`` (``--grid-origin=x,y,z`` when x is
negative, or argparse reads it as a flag).  Every command exits nonzero with a
message on a validation failure and writes its outputs atomically (temp
file + rename), so nothing partial is left behind.
"""
from __future__ import annotations

import argparse
import json
import sys
import time

import numpy as np


def _floats(s: str, n: int | None = None) -> tuple:
    v = tuple(float(x) for x in s.split(","))
    if n is not None and len(v) != n:
        raise argparse.ArgumentTypeError(f"expected {n} comma-separated numbers")
    return v


def _ints(s: str, n: int | None = None) -> tuple:
    v = tuple(int(x) for x in s.split(","))
    if n is not None and len(v) != n:
        raise argparse.ArgumentTypeError(f"expected {n} comma-separated integers")
    return v


def _grid_flags(p: argparse.ArgumentParser) -> None:
    p.add_argument("--grid-origin", type=lambda s: _floats(s, 3), default=(-40.0, -40.0, -1.0))
    p.add_argument("--grid-dims", type=lambda s: _ints(s, 3), default=(200, 200, 16))
    p.add_argument("--resolution", type=float, default=0.4)


def _spec(a):
    from .voxelize import VoxelGridSpec
    return VoxelGridSpec(a.grid_origin, a.grid_dims, a.resolution)


def _cfg(a):
    from .voxelize import VoxelizeConfig
    return VoxelizeConfig(tau=a.tau, neighborhood_radius=a.neighborhood, precision=a.precision)


def _emit(a, report: dict, text_lines: list[str]) -> None:
    if a.format == "json":
        print(json.dumps(report))
    else:
        print("\n".join(text_lines))


def cmd_gen_scene(a) -> int:
    from . import scenefile
    from .core import ClassTable
    from .scenegen import gen_frames
    if a.n < 0:
        raise ValueError("--n must be >= 0")
    spec = _spec(a)
    classes = ClassTable.numbered(a.classes)
    b = gen_frames(a.seed, 1, a.n, a.classes, origin=spec.origin, dims=spec.dims,
                   resolution=spec.resolution)
    scenefile.write(a.out, b, classes)
    _emit(a, {"command": "gen-scene", "out": a.out, "n": a.n, "classes": a.classes,
              "seed": a.seed}, [f"wrote {a.n} primitives to {a.out}"])
    return 0


def _n_prims(batch) -> int:
    return batch.n_prims if batch.n_valid is None else int(np.asarray(batch.n_valid)[0])


def _voxelize_scene(batch, classes, spec, cfg, truncate=True):
    """One timed voxelize of the scene: inputs already on the device, output
    grids preallocated, after one warm-up call (library load, workspace)."""
    import torch
    from .voxelize import Voxelizer
    vox = Voxelizer(spec, cfg, len(classes), classes.free_index, truncate=truncate)
    db = vox.to_device(batch)
    res = vox.alloc(1, dense=True)
    vox(db, dense=True, out=res)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = vox(db, dense=True, out=res)
    torch.cuda.synchronize()
    return r, (time.perf_counter() - t0) * 1e3, vox


def cmd_voxelize(a) -> int:
    from . import scenefile, sqoc
    from .voxelize import labels_to_host
    batch, classes = scenefile.read(a.scene)
    spec, cfg = _spec(a), _cfg(a)
    if not (1 <= len(classes) <= 255):
        raise ValueError("SQOC stores 1..255 classes")
    r, ms, _ = _voxelize_scene(batch, classes, spec, cfg)
    lab = labels_to_host(r.labels[0].cpu().numpy(), r.free_code, classes.free_index)
    vo = r.v_o[0].cpu().numpy() if a.vo else None
    sqoc.write(a.out, spec.dims, spec.origin, spec.resolution, len(classes), lab,
               classes.free_index, vo)
    occ = int(np.count_nonzero(r.labels[0].cpu().numpy() != r.free_code))
    n = _n_prims(batch)
    rep = {"command": "voxelize", "out": a.out, "dims": list(spec.dims),
           "resolution": spec.resolution, "n_prims": n, "pairs": r.n_pairs,
           "occupied_voxels": occ, "voxelize_ms": ms}
    lines = [f"voxelized {n} primitives -> {a.out} ({spec.dims[0]}x{spec.dims[1]}x"
             f"{spec.dims[2]} @ {spec.resolution} m), {occ} occupied voxels, {ms:.3f} ms"]
    if a.oracle:
        bf, ms_bf, _ = _voxelize_scene(batch, classes, spec, cfg, truncate=False)
        dvo = float((bf.v_o.double() - r.v_o.double()).abs().max().item())
        mism = float((bf.labels != r.labels).double().mean().item())
        rep.update({"oracle_ms": ms_bf, "max_abs_dvo": dvo, "label_mismatch_rate": mism})
        lines.append(f"oracle (voxelize_bruteforce): {ms_bf:.3f} ms, max |dv_o| = {dvo:.3e}, "
                     f"label mismatch rate {mism:.3e}")
    _emit(a, rep, lines)
    return 0


def _grid_of(g):
    """SqocGrid -> SemanticGrid (classes numbered, free = C)."""
    from .core import ClassTable
    from .voxelize import SemanticGrid, VoxelGridSpec
    spec = VoxelGridSpec(g.origin, g.dims, g.resolution)
    C = g.n_classes
    lab = np.where(g.labels == 255, C, g.labels).astype(np.int64)
    return SemanticGrid(lab.transpose(2, 1, 0), spec, ClassTable.numbered(C))


def cmd_metrics(a) -> int:
    from . import sqoc
    from .metrics import miou, ray_iou, voxel_iou
    p, g = _grid_of(sqoc.read(a.pred)), _grid_of(sqoc.read(a.gt))
    if tuple(p.spec.dims) != tuple(g.spec.dims):
        raise ValueError(f"dimension mismatch: {p.spec.dims} vs {g.spec.dims}")
    if len(p.classes) != len(g.classes):
        raise ValueError("class counts differ")
    iou = voxel_iou(p, g)
    per, m = miou(p, g)
    rays = ray_iou(p, g, thresholds=a.thresholds)
    rep = {"command": "metrics", "iou": iou, "miou": m,
           "per_class_iou": [None if not np.isfinite(x) else float(x) for x in per],
           "rayiou": rays}
    lines = [f"IoU {iou:.6f}", f"mIoU {m:.6f}",
             "per-class IoU " + " ".join(f"{x:.4f}" for x in per),
             "RayIoU " + json.dumps(rays)]
    _emit(a, rep, lines)
    return 0


def cmd_bench(a) -> int:
    import torch
    from . import scenefile
    batch, classes = scenefile.read(a.scene)
    spec, cfg = _spec(a), _cfg(a)
    if a.repetitions < 1:
        raise ValueError("--repetitions must be >= 1")
    out = {}
    for name, truncate in (("voxelize", True), ("oracle", False)):
        r, _, vox = _voxelize_scene(batch, classes, spec, cfg, truncate)
        db = vox.to_device(batch)
        res = r
        ts = []
        for _ in range(a.repetitions):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            vox(db, dense=True, out=res)
            torch.cuda.synchronize()
            ts.append((time.perf_counter() - t0) * 1e3)
        out[name] = {f"p{q}": float(np.percentile(ts, q)) for q in (10, 50, 90)}
    speedup = out["oracle"]["p50"] / out["voxelize"]["p50"]
    rep = {"command": "bench", "scene": a.scene, "n_prims": _n_prims(batch),
           "repetitions": a.repetitions, "wall_ms": out, "speedup_vs_oracle": speedup}
    lines = [f"{k}: p10 {v['p10']:.3f} ms  p50 {v['p50']:.3f} ms  p90 {v['p90']:.3f} ms"
             for k, v in out.items()] + [f"fast-vs-oracle speed-up {speedup:.1f}x"]
    _emit(a, rep, lines)
    return 0


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="sqocc", description=__doc__.split("\n\n")[0])
    sub = ap.add_subparsers(dest="command", required=True)
    g = sub.add_parser("gen-scene", help="seeded synthetic SceneFile (SPEC.md:594-597)")
    g.add_argument("--seed", type=int, required=True)
    g.add_argument("--n", type=int, required=True)
    g.add_argument("--classes", type=int, default=18)
    g.add_argument("--out", required=True)
    _grid_flags(g)
    g.set_defaults(run=cmd_gen_scene)
    for name, fn, hlp in (("voxelize", cmd_voxelize, "SceneFile -> SQOC grid (SPEC.md:576-581)"),
                          ("bench", cmd_bench, "voxelize timing (SPEC.md:589-592)")):
        p = sub.add_parser(name, help=hlp)
        p.add_argument("--scene", required=True)
        _grid_flags(p)
        p.add_argument("--tau", type=float, default=0.01)
        p.add_argument("--neighborhood", type=int, default=5)
        p.add_argument("--precision", choices=("strict", "fast"), default="strict")
        if name == "voxelize":
            p.add_argument("--out", required=True)
            p.add_argument("--oracle", action="store_true")
            p.add_argument("--vo", action="store_true", help="also store the f32 v_o block")
        else:
            p.add_argument("--repetitions", type=int, default=20)
        p.set_defaults(run=fn)
    m = sub.add_parser("metrics", help="IoU / mIoU / RayIoU of two SQOC grids (SPEC.md:586)")
    m.add_argument("--pred", required=True)
    m.add_argument("--gt", required=True)
    m.add_argument("--thresholds", type=_floats, default=(1.0, 2.0, 4.0))
    m.set_defaults(run=cmd_metrics)
    for p in (g, m, *(sub.choices[k] for k in ("voxelize", "bench"))):
        p.add_argument("--format", choices=("json", "text"), default="text")
    return ap


def main(argv=None) -> int:
    ap = build_parser()
    a = ap.parse_args(argv)
    try:
        return a.run(a)
    except (ValueError, OSError, RuntimeError) as e:
        print(f"sqocc {a.command}: error: {e}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
