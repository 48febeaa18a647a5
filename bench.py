#!/usr/bin/env python
"""bench.py — voxelized frames/s of the B200 superquadric voxelizer.

Workload (BASELINE.json config 2): synthetic frames of 2,000 superquadrics on
the Occ3D grid 200x200x16 @0.4 m, 18 classes, tau 0.01, N=5 window, seeded
generator of paper_2511_17361_b200/scenegen.py.  One step = one batch of
--frames-per-step frames (default 100) through the whole path: prep ->
scan -> emit -> radix sort -> evaluate+finalize (labels + dense v_o/v_c
written to HBM) -> confusion counts against ground-truth labels; for N > 1
the int64 confusion counts are all-reduced over NCCL inside the timed region.
Frames are sharded across ranks (weak scaling: each rank runs the same number
of frames per step).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Prints one JSON line on rank 0.  --impl reference times the CPU FP64 oracle
(oracle/, the reference's algorithm restated in C, all host threads) on a
bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "voxelized frames/sec (200×200×16, 18 cls, 2k SQs) at 1/2/4/8 B200; % FP32 roofline"
UNIT = "frames/s"
MUFU_PER_PAIR = 9      # 4 lg2 + 5 ex2 per (primitive, voxel) pair, SURVEY.md §8d
FP32_PER_PAIR = 40     # ~21 + (C+1) FP32-pipe instructions at C = 18, SURVEY.md §8d


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", type=int, choices=[1, 2, 3, 4], default=2,
                    help="BASELINE.json configs: 1 = 256 SQs, 2 = 2k SQs (headline), "
                         "3 = 4k SQs with eps in [0.1, 2], 4 = 8k SQs on 400x400x32 @0.2 m")
    ap.add_argument("--frames-per-step", type=int, default=None)
    ap.add_argument("--n-prims", type=int, default=None)
    ap.add_argument("--classes", type=int, default=18)
    ap.add_argument("--precision", choices=["strict", "fast"], default="strict")
    ap.add_argument("--seed", type=int, default=20251117)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    a = ap.parse_args()
    w = WORKLOADS[a.config]
    a.n_prims = a.n_prims or w["n_prims"]
    a.frames_per_step = a.frames_per_step or w["frames_per_step"]
    a.grid = dict(origin=w["origin"], dims=w["dims"], resolution=w["resolution"])
    a.gen = dict(a.grid, emin=w["emin"])
    return a


WORKLOADS = {
    1: dict(n_prims=256, frames_per_step=100, origin=(-40.0, -40.0, -1.0), dims=(200, 200, 16),
            resolution=0.4, emin=0.2),
    2: dict(n_prims=2000, frames_per_step=100, origin=(-40.0, -40.0, -1.0), dims=(200, 200, 16),
            resolution=0.4, emin=0.2),
    3: dict(n_prims=4000, frames_per_step=50, origin=(-40.0, -40.0, -1.0), dims=(200, 200, 16),
            resolution=0.4, emin=0.1),
    4: dict(n_prims=8000, frames_per_step=10, origin=(-40.0, -40.0, -1.0), dims=(400, 400, 32),
            resolution=0.2, emin=0.2),
}


def workload_config(a, world):
    d = a.grid["dims"]
    return {"workload": f"config{a.config}: synthetic frames x {a.n_prims} SQs, grid "
                        f"{d[0]}x{d[1]}x{d[2]} @{a.grid['resolution']} m, {a.classes} classes, "
                        f"tau 0.01, N=5 window, logit-sum, precision {a.precision}",
            "frames_per_step": a.frames_per_step, "frames_per_rank": a.frames_per_step * a.steps,
            "n_prims": a.n_prims, "grid": list(d), "resolution": a.grid["resolution"],
            "classes": a.classes, "generator": "scenegen.gen_frames (SPEC.md:594-597), seed "
                                               f"{a.seed}+frame; s~U[0.2,4], "
                                               f"eps~U[{a.gen['emin']},2]",
            "outputs": "labels u8 + v_o f32 + v_c f32 written per frame; confusion vs gt",
            "l2": "not flushed explicitly: each step writes "
                  f"{a.frames_per_step * d[0] * d[1] * d[2] * (5 + 4 * a.classes) / 1e9:.1f} GB "
                  "of outputs (>> 126 MB L2)",
            "parallelism": f"frame-sharded x{world} (no data-path collective; int64 confusion "
                           "all-reduce over NCCL)"}


# ---------------------------------------------------------------------------
# clocks during the timed region (B200_PROFILING.md recipe)
# ---------------------------------------------------------------------------

class ClockSampler:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-i", str(self.idx), "-lms", "50"], stdout=open(self.path, "w"),
                stderr=subprocess.DEVNULL)
            time.sleep(0.25)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.1)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        rows = []
        try:
            for line in open(self.path):
                p = [x.strip() for x in line.split(",")]
                if len(p) >= 9 and p[1].replace(".", "").isdigit():
                    rows.append(p)
        except Exception:
            pass
        if self.path:
            os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[1]) for r in rows]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in rows for n, v in zip(names, r[5:9]) if v == "Active"})
        loaded = [s for s in sm if s > 0.5 * max(sm)] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": float(rows[0][2]),
                "power_w_max": max(float(r[3]) for r in rows if r[3].replace(".", "").isdigit())
                if any(r[3].replace(".", "").isdigit() for r in rows) else None,
                "samples": len(rows), "reasons": reasons}


# ---------------------------------------------------------------------------
# CPU legs (oracle: test/baseline infrastructure only)
# ---------------------------------------------------------------------------

def cpu_run(a, max_frames, budget_s, threads=None):
    """Time the FP64 oracle (all host threads, or `threads`) on frames of the
    same workload until budget_s elapses or max_frames frames are done.
    Returns (frames/s, frames, seconds, threads, pairs/s)."""
    from oracle import oracle as O
    from paper_2511_17361_b200.scenegen import gen_frames
    O.build()
    all_threads = O.threads()
    if threads is not None:
        O.set_threads(threads)
    else:
        threads = all_threads
    grid, cfg = O.Grid(**a.grid), O.Cfg()
    done, pairs, t_total = 0, 0, 0.0
    while done < max_frames and (t_total < budget_s or done == 0):
        b = O.Prims.of(gen_frames(a.seed, 1, a.n_prims, a.classes, first_frame=done, **a.gen))
        t0 = time.perf_counter()
        r = O.voxelize(b, grid, cfg)
        t_total += time.perf_counter() - t0
        pairs += r["n_pairs"]
        done += 1
    O.set_threads(all_threads)
    return done / t_total, done, t_total, threads, pairs / t_total


def run_reference(a, rank, world):
    if rank != 0:
        return
    from paper_2511_17361_b200.scenegen import gen_frames
    from oracle import oracle as O
    O.build()
    grid, cfg = O.Grid(**a.grid), O.Cfg()
    frames = [O.Prims.of(gen_frames(a.seed, 1, a.n_prims, a.classes, first_frame=k, **a.gen))
              for k in range(a.warmup + a.steps)]
    for k in range(a.warmup):
        O.voxelize(frames[k], grid, cfg)
    t0 = time.perf_counter()
    pairs = 0
    for k in range(a.steps):
        pairs += O.voxelize(frames[a.warmup + k], grid, cfg)["n_pairs"]
    dt = time.perf_counter() - t0
    value = a.steps / dt
    line = {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference",
            "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
            "ms_per_step": 1e3 * dt / a.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            # the B200 arm's config verbatim (same workload, metric and unit);
            # each step times a bounded sample of it, one frame of the step's
            # batch (frames/s is a rate, so the sample size cancels), stated in
            # "sample" and cpu_baseline.sample
            "config": workload_config(a, world),
            "sample": f"1 frame of each {a.frames_per_step}-frame step ({a.steps} timed frames)",
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": O.threads(), "kind": "port",
                             "sample": f"{a.steps} frames (1 per step) of the config-{a.config} "
                                       "workload, "
                                       f"FP64 C oracle, OpenMP {O.threads()} threads; "
                                       f"{pairs / dt:.3e} pairs/s"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU leg
# ---------------------------------------------------------------------------

def run_ours(a, rank, world, local_rank):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2511_17361_b200 as P
    from paper_2511_17361_b200 import _lib
    from paper_2511_17361_b200.metrics import confusion_matrix
    from paper_2511_17361_b200.scenegen import gen_frames, jitter

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    spec = P.VoxelGridSpec(**a.grid)
    cfg = P.VoxelizeConfig(precision=a.precision)
    C, B, K, W = a.classes, a.frames_per_step, a.steps, a.warmup
    vox = P.Voxelizer(spec, cfg, C)
    n_batches = K
    first = rank * n_batches * B  # disjoint frames per rank (weak scaling)

    # ---- synthetic inputs (host, seeded) + ground truth (untimed) ----
    host_batches = [gen_frames(a.seed, B, a.n_prims, C, first_frame=first + k * B, **a.gen)
                    for k in range(n_batches)]
    dev_batches = [vox.to_device(b) for b in host_batches]
    gt = []
    for k, b in enumerate(host_batches):
        r = vox(jitter(b, seed=a.seed + 7919 + first + k), dense=False)
        gt.append(r.labels.clone())
    out = vox.alloc(B, dense=True)
    K1 = C + 1
    cm = torch.zeros((K1, K1), dtype=torch.int64, device=dev)
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- measured pipe peaks (roofline denominators) ----
    mufu_peak = _lib.microbench(0)
    ffma_peak = _lib.microbench(1)

    # two output slots: consecutive steps alternate CUDA streams, so the
    # binning of step k+1 overlaps the evaluation of step k (Voxelizer.run_many)
    outs = [out, vox.alloc(B, dense=True)]
    pairs_box = [0]

    entries_box = [0]

    def conf(k, r):
        pairs_box[0] += r.n_pairs
        entries_box[0] += r.n_entries
        confusion_matrix(r.labels, gt[k % n_batches], C, out=cm)

    # ---- warm-up ----
    vox.run_many([dev_batches[k % n_batches] for k in range(W)], outs, on_device=conf)
    barrier()

    # ---- timed: device-resident inputs ----
    cm.zero_()
    stats = torch.zeros(2, dtype=torch.int64, device=dev)  # evaluator MUFU ops, pairs
    _lib.stats_attach(stats)
    _lib.profile_enable(True)
    _lib.profile_read(reset=True)
    n_launch0 = _lib.launch_count()
    pairs = 0
    entries_box[0] = 0
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        barrier()
        ev0.record(stream)
        pairs_box[0] = 0
        vox.run_many([dev_batches[k % n_batches] for k in range(K)], outs, on_device=conf)
        pairs = pairs_box[0]
        if world > 1:
            dist.all_reduce(cm, op=dist.ReduceOp.SUM)
        ev1.record(stream)
        barrier()
    clocks = clk.summary()
    _lib.stats_attach(None)
    issued_mufu, eval_pairs = (int(v) for v in stats.cpu().tolist())
    launches = _lib.launch_count() - n_launch0
    prof = _lib.profile_read(reset=True)
    _lib.profile_enable(False)
    dt = max_over_ranks(ev0.elapsed_time(ev1) * 1e-3)
    frames_total = world * K * B
    value = frames_total / dt
    pairs_total = max_over_ranks(float(pairs))  # identical workload shape per rank

    def _peaks():
        try:
            return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        except Exception:
            return {}

    def hbm_roof(bytes_per_launch, secs):
        pk = _peaks().get("hbm_gbs")
        ach = bytes_per_launch / secs / 1e9
        return {"achieved": ach, "peak": pk, "unit": "GB/s", "frac": ach / pk if pk else None,
                "algorithmic": "labels u8 + v_o f32 + v_c f32 written per voxel",
                "peak_source": "MEASURED_PEAKS.json hbm_gbs" if pk else None}

    def tensor_roof(pairs_per_launch, C, secs):
        # the class accumulation as a contraction: 2 (C+1) FLOP per pair, run as
        # 3xTF32 on tcgen05; TF32 dense peak = half the measured bf16 peak
        pk = _peaks().get("bf16_tflops")
        ach = pairs_per_launch * 2 * (C + 1) / secs / 1e12
        return {"achieved": ach, "peak": pk / 2 if pk else None, "unit": "TFLOP/s",
                "frac": ach / (pk / 2) if pk else None,
                "algorithmic": f"2 x {C + 1} FLOP per in-window pair (class sums + sigma)",
                "peak_source": "MEASURED_PEAKS.json bf16_tflops / 2 (tf32)" if pk else None}

    def evaluator_name(entries_per_tile):
        # the library's choice (sqv_eval_tc_impl.cuh launch_tc): dense batches
        # stream, sparse ones (< 64 entries per tile) run the chunk-staged
        # persistent kernel; SQV_EVAL / SQV_STREAM override it (A/B runs)
        if os.environ.get("SQV_EVAL") == "ffma":
            return "eval_kernel (FFMA, sqv_eval.cu)"
        st = os.environ.get("SQV_STREAM")
        stream = entries_per_tile >= 64 if st is None else st != "0"
        return ("eval_tcs_kernel (tcgen05, per-warp streaming, 4 warps per CTA; "
                "sqv_eval_tc_impl.cuh)" if stream else
                "eval_tc_kernel (tcgen05, chunk-staged; sqv_eval_tc_impl.cuh)")

    # roofline of the dominant kernel (eval_kernel): algorithmic MUFU ops per
    # launch / its CUDA-event duration inside the timed region
    # (the evaluator kernel alone: events between the block-mask kernel and the
    # end of evaluate + finalize on the evaluating stream)
    eval_s = prof["eval_kernel_ms"] * 1e-3 / max(prof["calls"], 1)
    pairs_per_launch = pairs / max(K, 1)
    achieved = pairs_per_launch * MUFU_PER_PAIR / eval_s
    traffic, traffic_src, sfu_busy = None, None, None
    try:  # DRAM bytes of the evaluator from the committed ncu --set full capture, per launch
        import glob
        ppath = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_eval_tc_ncu.json")))[-1]
        pj = json.load(open(ppath))
        traffic = (pj["dram_bytes_read"] + pj["dram_bytes_write"]) * B / pj["frames_per_launch"]
        traffic_src = (os.path.relpath(ppath, ROOT) +
                       f" (ncu {pj['frames_per_launch']}-frame launch, scaled to {B})")
        sfu_busy = {"frac": pj["xu_pct"] / 100.0, "issue_frac": pj["issue_pct"] / 100.0,
                    "source": os.path.relpath(ppath, ROOT),
                    "note": "MUFU ops actually issued (ncu sm__inst_executed_pipe_xu): frac "
                            "counts 9 MUFU for every in-window pair, the kernel issues 7 per "
                            "evaluated pair and skips warp blocks whose F exceeds the cull "
                            "threshold (< 2e-12 dropped per voxel), so frac can pass 1"}
    except Exception:
        pass
    roofline = {"bound": "sfu", "achieved": achieved / 1e9, "peak": mufu_peak / 1e9,
                "unit": "Gop/s (MUFU ex2/lg2)", "frac": achieved / mufu_peak, "traffic": traffic,
                "traffic_source": traffic_src, "sfu_busy_ncu": sfu_busy,
                "algorithmic_bytes_per_launch": B * spec.n_voxels * (1 + 4 + 4 * C),
                "kernel": evaluator_name(entries_box[0] / max(K * B * vox.tiles_per_frame, 1)),
                "algorithmic": f"{MUFU_PER_PAIR} MUFU per in-window (primitive, voxel) pair x "
                               f"{pairs_per_launch:.4e} pairs per launch",
                "eval_ms_per_launch": eval_s * 1e3,
                "eval_share_of_step": prof["eval_kernel_ms"] / max(1e-9, dt * 1e3),
                "stage_ms_per_step": {"masks_and_eval_ms": prof["eval_ms"] / max(prof["calls"], 1),
                                      "eval_kernel_ms": eval_s * 1e3},
                "stage_note": "CUDA-event spans on the evaluating stream: the block-mask kernel "
                              "+ the evaluator, and the evaluator alone (the roofline's time); "
                              "consecutive steps alternate two streams (binning of k+1 under "
                              "the evaluation of k), so the binning spans are not reported "
                              "(they contain the other stream's evaluation)",
                "peak_source": "sqv_microbench(MUFU) measured live on this GPU",
                "bound_note": "the field (powers, exps) is transcendental: the SFU pipe bounds "
                              "the evaluator; the contract's hbm and tensor rooflines of the "
                              "same kernel are below for comparison",
                "issued": {
                    "mufu_ops_per_launch": issued_mufu / max(K, 1),
                    "achieved": issued_mufu / max(K, 1) / eval_s / 1e9,
                    "frac": issued_mufu / max(K, 1) / eval_s / mufu_peak,
                    "evaluated_pairs_per_launch": eval_pairs / max(K, 1),
                    "evaluated_share_of_window_pairs": eval_pairs / max(pairs, 1),
                    "note": "MUFU ops the evaluators actually issue, counted live on the "
                            "device (sqv_stats_attach: per warp block run, 7 per voxel strict, "
                            "4 for accurate-log primitives, 6.5 fast), over the same eval time "
                            "and peak: the kernel-quality fraction; frac above counts the "
                            "algorithmic 9 per in-window pair"},
                "hbm": hbm_roof(B * spec.n_voxels * (1 + 4 + 4 * C), eval_s),
                "tensor": tensor_roof(pairs_per_launch, C, eval_s),
                "fp32_pipe": {"achieved_glanes": pairs_per_launch * FP32_PER_PAIR / eval_s / 1e9,
                              "peak_glanes": ffma_peak / 1e9,
                              "frac": pairs_per_launch * FP32_PER_PAIR / eval_s / ffma_peak}}

    # ---- e2e: public API from pinned host buffers, labels back to host ----
    e2e = None
    if not a.no_e2e:
        pinned = []
        for b in host_batches:
            f = {k: torch.from_numpy(np.ascontiguousarray(getattr(b, k))).pin_memory()
                 for k in P.PrimitiveBatch.FIELDS}
            pinned.append(P.PrimitiveBatch(**f))
        cm_host = torch.empty(cm.shape, dtype=torch.int64).pin_memory()
        h2d = sum(getattr(pinned[0], k).numel() * 8 for k in P.PrimitiveBatch.FIELDS)
        d2h = B * spec.n_voxels
        seq = [pinned[k % n_batches] for k in range(K)]
        labels_host = [torch.empty((B,) + tuple(out.labels.shape[1:]), dtype=torch.uint8)
                       .pin_memory() for _ in range(K)]

        def conf(k, res):
            confusion_matrix(res.labels, gt[k % n_batches], C, out=cm)

        vox.stream(seq[:2], dense=True, on_device=conf, labels_out=labels_host[:2])  # warm-up
        barrier()
        cm.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        t0 = time.perf_counter()
        e0.record(stream)
        vox.stream(seq, dense=True, on_device=conf, labels_out=labels_host)
        if world > 1:
            dist.all_reduce(cm, op=dist.ReduceOp.SUM)
        cm_host.copy_(cm, non_blocking=True)
        e1.record(stream)
        barrier()
        wall = time.perf_counter() - t0
        dt_e2e = max_over_ranks(e0.elapsed_time(e1) * 1e-3)
        e2e = {"value": frames_total / dt_e2e, "unit": UNIT, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "wall_s": max_over_ranks(wall),
               "path": "Voxelizer.stream over pinned host PrimitiveBatches: H2D of step k+1 and "
                       "D2H of step k-1 labels on copy streams overlap step k; confusion on "
                       "device; int64 counts read back at the end"}

    # ---- CPU baseline (rank 0, N = 1 only) ----
    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        fps, nfr, secs, thr, pps = cpu_run(a, 8, a.cpu_seconds)
        fps1, nfr1, secs1, _, pps1 = cpu_run(a, 1, 0.0, threads=1)
        cpu = {"value": fps, "unit": UNIT, "cores": thr, "kind": "port",
               "sample": f"{nfr} frames of the config-2 workload in {secs:.1f} s, FP64 C oracle "
                         f"(oracle/sqv_oracle.c), OpenMP {thr} threads; {pps:.3e} pairs/s",
               "single_thread": {"value": fps1, "unit": UNIT, "pairs_per_s": pps1,
                                 "sample": f"{nfr1} frame in {secs1:.1f} s, 1 thread"}}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K,
                "warmup": W, "ms_per_step": 1e3 * dt / K, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f32 (fp64 prep)",
                "data": "synthetic", "config": workload_config(a, world),
                "pairs_per_s": world * pairs_total / dt, "gpu_launches": launches,
                "roofline": roofline, "clocks": clocks, "e2e": e2e, "cpu_baseline": cpu,
                "confusion_total": int(cm.sum().item())}
        print(json.dumps(line), flush=True)


def main():
    a = parse()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if a.impl == "reference":
        run_reference(a, rank, world)
        return
    import torch
    import torch.distributed as dist
    if world > 1:
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        run_ours(a, rank, world, local_rank)
    finally:
        if world > 1:
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
