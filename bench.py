#!/usr/bin/env python
"""bench.py -- THIIM sweep throughput (MLUP/s) on B200, per the driver contract.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl native|reference]
                    [--config c0..c4]

Workload: the largest single-GPU BASELINE.json config, configs[2] (512^3 grid,
complex128, 200 THIIM iterations -- H half-step then E half-step in the
reference's step_reference order -- per bench step; fields U[-1,1]^2, 28
coefficient arrays uniform in |z|<=0.45, seed 1, zero ghosts) at N=1, and
configs[4] (a 1024x1024x128 z-slab per GPU, 100 iterations, weak scaling) at
N>1.  One bench "step" = one full run of that config.

  value   MLUP/s with the problem resident in HBM (device time, CUDA events on
          the launching stream), max over ranks.
  e2e     same metric through the public API, every step's inputs uploaded
          from pinned host memory and its 12 result fields downloaded: the
          faster of a stream of problems (run_gpu_batch, one problem per step,
          <= 20; at configs[2] two TBLOCK-in-place contexts so uploads overlap
          sweeps) and the one-problem call sequence (run_gpu); both reported.
  roofline  dominant kernel vs measured HBM.
  cpu_baseline  the reference's own run_naive (oracle/_ref, compiled from
          /root/reference unmodified) on the host cores, bounded sample.

--impl reference runs the reference CPU implementation alone (rank 0 only) on a
bounded sample of the same config; its inputs come from the oracle's generator
(oracle/), never from this package.  Multi-rank (torchrun): weak scaling, rank r
owns z-slab r of the global grid (paper_1510_05218_b200/distributed.py).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SEED = 1
# BASELINE.json configs; the default bench line is configs[2] (N=1), configs[4] per rank (N>1)
CONFIGS = {
    "c0": ((64, 64, 64), 50, 0, "configs[0]: 64^3 grid, 50 THIIM iterations"),
    "c1": ((256, 256, 256), 100, 0, "configs[1]: 256x256x256 grid, 100 THIIM iterations"),
    "c2": ((512, 512, 512), 200, 0, "configs[2]: 512^3 grid, 200 THIIM iterations"),
    "c3": ((1024, 1024, 256), 200, 1, "configs[3]: layered thin-film 1024x1024x256, 200 THIIM "
                                      "iterations, 6 z-layers, +-8-cell seeded interfaces"),
    "c4": ((1024, 1024, 128), 100, 0, "configs[4]: weak-scaling slab 1024x1024x128 per GPU, 100 "
                                      "THIIM iterations"),
}
DEFAULT_SINGLE, DEFAULT_MULTI = "c2", "c4"
GRID, ITERS, KIND, _DESC = CONFIGS[DEFAULT_SINGLE]
WORKLOAD = (_DESC + " (H then E half-step) per bench step, complex128, fields U[-1,1], "
            "coeffs |c|<=0.45, seed 1, zero halo")
METRIC = "MLUP/s (double-complex E+H update) at N B200; % of HBM roofline"


def default_config(world: int) -> str:
    """configs[2] (the largest single-GPU config) at N=1, configs[4] (the
    weak-scaling slab per GPU) at N>1."""
    return DEFAULT_SINGLE if world == 1 else DEFAULT_MULTI


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            j = json.load(f)
        return float(j.get("hbm_gbs", 6650.0)), "measured"
    return 6650.0, "fallback"


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


class Clocks:
    """nvidia-smi sampler running during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), "--query-gpu=" + self.Q,
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.result = {"sm_mhz": None, "sm_max_mhz": None, "reasons": []}
        if not self.proc:
            return
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out = ""
        sm, pw, mx, reasons = [], [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        post = False
        if not out.strip():  # timed region shorter than the sampler's first tick
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.device), "--query-gpu=" + self.Q,
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=30).stdout
                post = True
            except Exception:
                out = ""
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            try:
                pw.append(float(f[3]))
            except ValueError:
                pass
            for n, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        if sm:
            self.result = {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx,
                           "reasons": sorted(reasons), "samples": 0 if post else len(sm),
                           "power_w": float(np.median(pw)) if pw else None}
            if post:
                self.result["note"] = "timed region shorter than one sampling tick: post-run sample"


def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def sample_grid(grid):
    """Bounded CPU sample of a config: its x-y plane, with the z extent cut so
    the sample holds about 2^25 cells (the whole grid when it is smaller)."""
    nx, ny, nz = grid
    return (nx, ny, max(8, min(nz, (1 << 25) // (nx * ny))))


def reference_engines_sample(grid, threads):
    """The reference's other CPU engines on the same sample: its
    spatially blocked sweep (block_y 8) and its multicore wavefront-diamond
    engine (the paper's temporal blocking; dw 8, bz 1, one thread per group),
    4 iterations each -- context for the naive baseline `value`."""
    from oracle import oracle as O  # cpu baseline leg only
    if not O.ref_available():
        return {}
    cells = grid[0] * grid[1] * grid[2]
    out = {}
    try:
        with O.RefState(grid) as r:
            r.generate(SEED, bool(KIND), threads)
            secs = r.run_spatial(4, 8, 0, threads)
            out["spatial_blocked_mlups"] = round(cells * 4 / secs / 1e6, 3)
            r.generate(SEED, bool(KIND), threads)
            secs, executed = r.run_mwd(4, 8, 1, 1, 1, 1, threads)
            out["mwd_mlups"] = round(cells * executed / secs / 1e6, 3)
        out["mwd_params"] = "dw 8, bz 1, shape 1x1x1, %d threads" % threads
        # the reference's own host triad (its `bandwidth` subcommand), SURVEY s8d
        out["host_triad_gbs"] = round(O.ref_measure_bandwidth(threads), 1)
    except Exception as e:  # report, never fail the bench line
        out["reference_engines_error"] = str(e)[:200]
    return out


class _CpuRef:
    """The reference's run_naive on a problem generated inside oracle/_ref
    (ref_shim.cpp: the seeded generator restated there, so only the reference
    library is loaded); the oracle's C port when oracle/_ref is absent."""

    def __init__(self, grid, threads):
        from oracle import oracle as O  # cpu baseline / reference arm only
        self.O, self.grid, self.threads = O, grid, threads
        self.kind = "reference" if O.ref_available() else "port"
        if self.kind == "reference":
            self.r = O.RefState(grid)
            self.r.generate(SEED, bool(KIND), threads)
        else:
            self.a = O.c_generate(grid, SEED, layered=bool(KIND))

    def run(self, iters):
        if self.kind == "reference":
            return self.r.run_naive(iters, self.threads)
        t0 = time.perf_counter()
        self.O.c_step(self.grid, self.a, iters, threads=self.threads)
        return time.perf_counter() - t0

    def close(self):
        if self.kind == "reference":
            self.r.close()


def reference_sample(grid, iters, threads):
    """Time the reference's run_naive (oracle/_ref) on the sample problem."""
    c = _CpuRef(grid, threads)
    secs = c.run(iters)
    c.close()
    return grid[0] * grid[1] * grid[2] * iters / secs / 1e6, c.kind


def run_reference_arm(args, world, rank):
    """The reference's own CPU path (oracle/_ref run_naive, all host threads)
    on a bounded sample of the bench config: the config's x-y planes, ~2^25
    cells, one THIIM iteration per step.  The problem is generated inside the
    reference library's shim (bitwise the product's generator,
    tests/test_oracle.py); this arm never imports or loads the product package."""
    if rank != 0:
        return
    threads = cpu_threads()
    sample_iters = 1
    grid = sample_grid(GRID)
    c = _CpuRef(grid, threads)
    vals = []
    for k in range(args.warmup + args.steps):
        secs = c.run(sample_iters)
        if k >= args.warmup:
            vals.append(secs)
    c.close()
    secs = sum(vals)
    cells = grid[0] * grid[1] * grid[2]
    v = cells * sample_iters * len(vals) / secs / 1e6
    sample = ("%dx%dx%d x %d iteration(s) per step (the config's x-y planes, z cut to a bounded "
              "sample), run_naive threads=%d, problem generated in oracle/_ref"
              % (grid + (sample_iters, threads)))
    line = {
        "impl": "reference", "metric": METRIC, "value": round(v, 3), "unit": "MLUP/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 * secs / max(1, len(vals)), 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "c128 (f64)", "data": "synthetic",
        "config": {"workload": WORKLOAD, "config": args.config, "grid": list(GRID),
                   "sample_grid": list(grid), "iterations_per_step": sample_iters,
                   "note": "reference run_naive on host cores; each step a bounded sample"},
        "cpu_baseline": {"value": round(v, 3), "unit": "MLUP/s", "cores": threads, "kind": c.kind,
                         "sample": sample},
        "e2e": {"value": round(v, 3), "unit": "MLUP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _roofline(P, dims, engine_ran, dev_secs, launches, table=False, iters_total=0, depth=2):
    """Roofline of the dominant kernel: one THIIM iteration (fused) or one
    half-step sweep (split) per launch over the rank's grid.  TBLOCK in place:
    one two-step pass (its sub-range launches + copy-back) is the unit."""
    hbm, peak_kind = load_peaks()
    per_launch_s = dev_secs / max(1, launches)
    if engine_ran == P.ENGINE_TBLOCK:
        # a TBLOCK pass (`depth` iterations) is one launch per round of <= 148
        # CTAs: the unit is the pass
        per_launch_s = dev_secs / max(1, iters_total / depth)
    if engine_ran == P.ENGINE_TBLOCK_INPLACE:
        per_launch_s = dev_secs / max(1, iters_total / 2)
        bytes_launch = 832.0 * dims.interior_cells()  # one pass, outputs shifted into the gap
        kname = "k_tblock_tm<15,6> sub-ranges (in place)"
    elif engine_ran == P.ENGINE_SPLIT:
        bytes_launch = 512.0 * dims.interior_cells()  # one half-step sweep: 32 x 16 B per cell
        kname = "k_split_h/k_split_e"
    elif table and engine_ran == P.ENGINE_TBLOCK:
        # one launch = two iterations: 24 fields x 16 B + 1 B material id per cell
        bytes_launch = 385.0 * dims.interior_cells()
        kname = "k_tblock_table<15,5>"
    elif table:
        bytes_launch = 385.0 * dims.interior_cells()  # 24 fields x 16 B + 1 B material id
        kname = "k_fused_table<15,5>"
    elif engine_ran == P.ENGINE_TBLOCK:
        # one pass = `depth` THIIM iterations: 832 B per cell = 832/depth B/LUP
        bytes_launch = 832.0 * dims.interior_cells()
        kname = "k_tblock3_tm<15,6>" if depth == 3 else "k_tblock_tm<15,6>"
    else:
        bytes_launch = 832.0 * dims.interior_cells()
        kname = "k_fused_tma<15,6>"
    achieved = bytes_launch / per_launch_s / 1e9
    # ncu DRAM bytes per launch of this kernel on this grid (profiles/traffic.json,
    # written by tools/summarize_ncu.py); null for a grid that was not captured
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        with open(tp) as f:
            traffic = json.load(f).get("%s@%dx%dx%d" % (kname, dims.nx, dims.ny, dims.nz))
    balance = (385.0 / (2 if engine_ran == P.ENGINE_TBLOCK else 1)) if table \
        else P.balance_model(engine_ran, depth if engine_ran == P.ENGINE_TBLOCK else 0)
    steps_per_launch = 2 if engine_ran in (P.ENGINE_TBLOCK, P.ENGINE_TBLOCK_INPLACE) else 1
    if engine_ran == P.ENGINE_TBLOCK and not table:
        steps_per_launch = depth
    if engine_ran == P.ENGINE_SPLIT:
        steps_per_launch = 0.5
    return {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm, "unit": "GB/s",
            "frac": round(achieved / hbm, 4), "traffic": traffic, "kernel": kname,
            "algorithmic_bytes_per_launch": bytes_launch, "peak_kind": peak_kind,
            "bytes_per_lup_model": balance,
            "traffic_bytes_per_lup": (round(traffic / (dims.interior_cells() * steps_per_launch), 1)
                                      if traffic else None),
            "lup_roofline_mlups": round(hbm * 1e3 / balance, 1)}


def run_native(args, world, rank, local):
    import paper_1510_05218_b200 as P
    engine = {"auto": P.ENGINE_AUTO, "split": P.ENGINE_SPLIT, "fused": P.ENGINE_FUSED,
              "tblock": P.ENGINE_TBLOCK, "tblock-inplace": P.ENGINE_TBLOCK_INPLACE}[args.engine]
    opts = P.GpuOptions(device=local if world > 1 else args.device, engine=engine,
                        tile_y=args.tile_y, z_chunk=args.z_chunk, schedule=args.schedule,
                        band=args.band, time_block=args.time_block,
                        coeff_layout=P.COEFF_TABLE if args.coeff == "table" else P.COEFF_FULL,
                        n_materials=6 if args.coeff == "table" else 0)
    iters = args.iters
    if world == 1:
        line = run_native_single(P, args, opts, iters)
    else:
        line = run_native_multi(P, args, opts, iters, world, rank, local)
    if line is None:
        return
    if world == 1 and not args.no_cpu_baseline:
        threads = cpu_threads()
        grid = sample_grid(GRID)
        v, kind = reference_sample(grid, 2, threads)
        line["cpu_baseline"] = {"value": round(v, 3), "unit": "MLUP/s", "cores": threads,
                                "kind": kind,
                                "sample": "reference run_naive (oracle/_ref, compiled unmodified), "
                                          "%dx%dx%d x 2 iterations, %d threads, problem "
                                          "generated in oracle/_ref" % (grid + (threads,))}
        line["cpu_baseline"].update(reference_engines_sample(grid, threads))
    print(json.dumps(line), flush=True)


def _line(P, args, world, dims_rank, engine_ran, dev_secs, launches, e2e, clk, extra_cfg):
    lups_step = dims_rank.interior_cells() * args.iters
    value = world * lups_step * args.steps / dev_secs / 1e6
    padded = dims_rank.padded_cells() * 16
    cfg = {"workload": WORKLOAD, "config": args.config, "coeff_layout": args.coeff,
           "grid_per_rank": [dims_rank.nx, dims_rank.ny, dims_rank.nz],
           "iterations_per_step": args.iters, "engine": P.ENGINE_NAMES.get(engine_ran),
           "parallelism": "z-slab x%d" % world if world > 1 else "single GPU",
           "l2": "inputs (%.1f GB state per GPU) larger than the 126 MB L2; no flush needed"
                 % (dims_rank.padded_cells() * (385 if args.coeff == "table" else
                                                640 if engine_ran in (P.ENGINE_SPLIT,
                                                                      P.ENGINE_TBLOCK_INPLACE)
                                                else 832) / 1e9)}
    cfg.update(extra_cfg)
    return {
        "metric": METRIC, "value": round(value, 2), "unit": "MLUP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 * dev_secs / args.steps, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "c128 (f64)", "data": "synthetic",
        "config": cfg,
        "e2e": {"value": round(e2e, 2) if e2e else None, "unit": "MLUP/s",
                "h2d_bytes_per_step": 40 * padded, "d2h_bytes_per_step": 12 * padded},
        "gpu_launches": launches,
        "roofline": _roofline(P, dims_rank, engine_ran, dev_secs, launches,
                              table=getattr(args, "coeff", "full") == "table",
                              iters_total=args.iters * args.steps,
                              depth=getattr(args, "depth_ran", 2)),
        "clocks": clk.result,
    }


def _device_bytes(device: int) -> int:
    """Total memory of the GPU (bytes)."""
    import torch
    return torch.cuda.get_device_properties(device).total_memory


def host_available_bytes() -> int:
    try:
        with open("/proc/meminfo") as f:
            for line in f:
                if line.startswith("MemAvailable:"):
                    return int(line.split()[1]) * 1024
    except OSError:
        pass
    return 0


def e2e_skip_reason(args, dims):
    """Why the host-memory e2e leg cannot run for this configuration, or None."""
    if args.coeff == "table":
        return ("table layout: its inputs (material ids + table) are this engine's own format, "
                "generated on the device; e2e is measured on the reference layout")
    need = 52 * dims.padded_cells() * 16  # 40 input arrays + 12 result fields, pinned
    avail = host_available_bytes()
    if avail and need > 0.8 * avail:
        return "host RAM: %.0f GB of pinned inputs/outputs, %.0f GB available" % (need / 1e9,
                                                                               avail / 1e9)
    return None


def run_native_single(P, args, opts, iters):
    dims = P.GridDims(*GRID)
    eng = P.GpuEngine(dims, opts)
    eng.generate(KIND, SEED)
    for _ in range(args.warmup):
        eng.step(iters)
    dev_secs, launches = 0.0, 0
    with Clocks(opts.device) as clk:
        for _ in range(args.steps):
            st = eng.step(iters)  # CUDA events on the launching stream, inside the library
            dev_secs += st.seconds
            launches += st.kernel_launches
    engine_ran = st.engine
    if engine_ran == P.ENGINE_TBLOCK and args.coeff != "table" and st.balance_model > 0:
        args.depth_ran = int(round(832.0 / st.balance_model))  # time-block depth that ran
    eng.close()

    # e2e: the public API a user calls, with every step's inputs copied from
    # pinned host memory and its 12 result fields copied back.  Headline: the
    # pipelined stream API (run_gpu_batch: step i uploads while i-1 computes and
    # i-2 downloads, all inside one timed call incl. context create/destroy).
    # Beside it the one-problem call sequence (create, upload, step, download,
    # destroy), serial, with its phases.
    e2e = None
    e2e_extra = {}
    skip = e2e_skip_reason(args, dims)
    if skip:
        e2e_extra = {"skipped": skip}
    if not args.no_e2e and not skip:
        host = P.generate_problem(dims, KIND, SEED)
        out = [np.zeros_like(a) for a in host.fields]
        pinned = host.arrays + out
        for a in pinned:
            P.lib().thiim_gpu_pin_host(a.ctypes.data, a.nbytes)
        # the stream overlaps problem i's upload with i-1's sweep when the
        # device holds >= 2 contexts: ping-pong TBLOCK (52 arrays) up to
        # configs[1]; at configs[2] it holds one, and the library's batch plan
        # runs two TBLOCK-in-place contexts (40 arrays + a gap each) instead
        stream = None
        if 2 * 40 * dims.padded_cells() * 16 < 0.97 * _device_bytes(opts.device):
            # untimed warm-up; 3 problems so the device pool already holds the
            # three contexts the timed call reuses
            P.run_gpu_batch([host] * 3, iters, opts, outputs=[out] * 3)
            nstream = min(args.steps, 20)  # bounded: ~2.5 s per configs[2] problem
            rep = P.run_gpu_batch([host] * nstream, iters, opts, outputs=[out] * nstream)
            stream = {
                "value": round(dims.interior_cells() * iters * nstream / rep.seconds / 1e6, 2),
                "api": "run_gpu_batch (thiim_gpu_run_batch), depth %d, one problem per step, "
                       "%d steps" % (rep.depth, nstream),
                "depth": rep.depth,
                "engine": rep.engine,
                "call_ms": round(1e3 * rep.seconds, 1),
                "device_span_ms": round(1e3 * rep.device_seconds, 1),
                "device_ms_per_step": {
                    "upload": round(1e3 * rep.upload_seconds / nstream, 2),
                    "sweep": round(1e3 * rep.kernel_seconds / nstream, 2),
                    "download": round(1e3 * rep.download_seconds / nstream, 2)},
            }
        secs = 0.0
        phases = [0.0] * 5
        nser = max(1, min(args.steps, 3))
        for k in range(1 + nser):  # 1 untimed warm-up
            t = [time.perf_counter()]
            e = P.GpuEngine(dims, opts)
            t.append(time.perf_counter())
            e.upload(host)
            t.append(time.perf_counter())
            e.step(iters)
            t.append(time.perf_counter())
            e.download_fields(out)
            t.append(time.perf_counter())
            e.close()
            t.append(time.perf_counter())
            if k >= 1:
                secs += t[-1] - t[0]
                for j in range(5):
                    phases[j] += t[j + 1] - t[j]
        for a in pinned:
            P.lib().thiim_gpu_unpin_host(a.ctypes.data)
        del host, out, pinned
        serial = {
            "value": round(dims.interior_cells() * iters * nser / secs / 1e6, 2),
            "api": "run_gpu call sequence (create, upload, step, download, destroy), %d steps"
                   % nser,
            "phases_ms_per_step": dict(zip(["create", "upload", "step", "download", "destroy"],
                                           [round(1e3 * v / nser, 2) for v in phases])),
        }
        # headline: the faster of the two public-API paths (the stream overlaps
        # copies with sweeps when the device holds >= 2 contexts; with one it
        # cannot, and the plain call sequence is the better way to run)
        best = stream if stream and stream["value"] >= serial["value"] else serial
        e2e = best["value"]
        e2e_extra = {"api": best["api"], "serial": serial}
        if stream:
            e2e_extra["stream"] = stream
        else:
            e2e_extra["stream"] = "not run: the device holds one context of this size"
    line = _line(P, args, 1, dims, engine_ran, dev_secs, launches, e2e, clk, {})
    line["e2e"].update(e2e_extra)
    return line


def run_native_multi(P, args, opts, iters, world, rank, local):
    """Weak scaling: rank r owns z-slab r (the config's grid, configs[4] by
    default: 1024x1024x128) of an nx x ny x (nz*N) grid; TBLOCK slabs store
    their boundary planes into the neighbours' halos (CUDA IPC peer stores)."""
    import torch
    import torch.distributed as dist
    from paper_1510_05218_b200 import distributed as D
    # THIIM_DIST_BACKEND=gloo + THIIM_SAME_DEVICE=1 run every rank on cuda:0 with
    # host-staged halos (test mode for hosts with one GPU); default NCCL, GPU = local rank
    backend = os.environ.get("THIIM_DIST_BACKEND", "nccl")
    if os.environ.get("THIIM_SAME_DEVICE") == "1":
        local = 0
        opts.device = 0
    torch.cuda.set_device(local)
    dist.init_process_group(backend)
    gdims = P.GridDims(GRID[0], GRID[1], GRID[2] * world)
    z0, z1 = D.slab_bounds(gdims.nz, world, rank)
    ex = D.HaloExchanger(rank, world)
    # THIIM_PEER_STORES=0: exchange halos with torch.distributed after every pass
    want_peer = os.environ.get("THIIM_PEER_STORES", "1") != "0"

    def make_engine():
        e = D.SlabGpuEngine(gdims, z0, z1, opts)
        if want_peer:
            e.enable_peer_stores(rank, world)
        return e

    eng = make_engine()
    eng.generate(P.GEN_RANDOM, SEED)
    for _ in range(args.warmup):
        D.run_distributed(eng, iters, ex)

    def timed(fn):
        dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out = fn()
        eng.sync()
        torch.cuda.synchronize()
        e1.record()
        e1.synchronize()
        dev = "cuda" if backend == "nccl" else "cpu"
        t = torch.tensor([e0.elapsed_time(e1) * 1e-3], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item()), out

    launches = 0
    with Clocks(local) as clk:
        dev_secs, stats = timed(lambda: [D.run_distributed(eng, iters, ex)
                                         for _ in range(args.steps)])
    launches = sum(s["kernel_launches"] for s in stats)
    halo = sum(s["halo_bytes_sent"] for s in stats)
    engine_ran, period, peer = eng.engine, eng.exchange_period, eng.peer_stores
    ordered = getattr(eng, "device_ordered", False)
    eng.close()

    # the same per-rank workload on one GPU (a whole-z context of the rank's
    # grid, rank 0 alone, device time): the N=1 point of this config's weak
    # scaling (the N=1 bench line is configs[2]); the driver computes any
    # efficiency from it
    n1 = None
    if not args.no_n1_base:
        dist.barrier()
        if rank == 0:
            e1 = P.GpuEngine(P.GridDims(*GRID), opts)
            e1.generate(P.GEN_RANDOM, SEED)
            e1.step(iters)  # warm-up
            k1 = max(1, min(args.steps, 3))
            secs1 = sum(e1.step(iters).seconds for _ in range(k1))
            e1.close()
            n1 = {"value": round(P.GridDims(*GRID).interior_cells() * iters * k1 / secs1 / 1e6, 2),
                  "unit": "MLUP/s", "steps": k1,
                  "what": "the per-rank grid as one whole-z context on one GPU (rank 0, device time)"}
        dist.barrier()

    e2e = None
    # every local rank pins its slab's 40 arrays on the host: skip the leg if
    # the node's RAM does not hold all of them (decided identically by all ranks)
    rank_bytes = 40 * (GRID[0] + 2) * (GRID[1] + 2) * (GRID[2] + 4) * 16
    local_ranks = int(os.environ.get("LOCAL_WORLD_SIZE", str(world)))
    avail = host_available_bytes()
    e2e_skip = (avail and local_ranks * rank_bytes > 0.7 * avail)
    if e2e_skip:
        flag = torch.tensor([1], dtype=torch.int32, device="cuda" if backend == "nccl" else "cpu")
    else:
        flag = torch.tensor([0], dtype=torch.int32, device="cuda" if backend == "nccl" else "cpu")
    dist.all_reduce(flag, op=dist.ReduceOp.MAX)
    e2e_skip = bool(flag.item())
    if not args.no_e2e and not e2e_skip:
        eng = make_engine()
        host = eng.local_host_problem(P.GEN_RANDOM, SEED)
        for a in host:
            P.lib().thiim_gpu_pin_host(a.ctypes.data, a.nbytes)

        n_e2e = max(1, min(args.steps, 3))

        def e2e_run():
            for _ in range(n_e2e):
                eng.upload_local(host)
                D.run_distributed(eng, iters, ex)
                eng.download_local(host)
        e2e_run_secs, _ = timed(e2e_run)
        for a in host:
            P.lib().thiim_gpu_unpin_host(a.ctypes.data)
        eng.close()
        e2e = world * P.GridDims(*GRID).interior_cells() * iters * n_e2e / e2e_run_secs / 1e6
    if args.check:
        # decomposed run vs one oracle run of the global grid, gathered on rank 0
        eng = make_engine()
        host = eng.local_host_problem(KIND, SEED)
        eng.upload_local(host)
        D.run_distributed(eng, args.check, ex)
        eng.download_local(host)
        mine = np.stack([eng.owned_planes(host, k) for k in range(12)])
        eng.close()
        pxy = (gdims.nx + 2) * (gdims.ny + 2)
        parts = [None] * world
        dist.all_gather_object(parts, (z0, z1, mine))
        if rank == 0:
            from oracle import oracle as O  # parity check only
            ref = P.generate_problem(gdims, KIND, SEED)
            O.c_step((gdims.nx, gdims.ny, gdims.nz), ref.arrays, args.check, threads=cpu_threads())
            ok = all(np.array_equal(m[k].view(np.uint64),
                                    ref.arrays[k][(a + 1) * pxy:(b + 1) * pxy].view(np.uint64))
                     for a, b, m in parts for k in range(12))
            print(json.dumps({"check": "z-slab decomposition vs oracle", "ranks": world,
                              "steps": args.check, "bitwise_equal": bool(ok)}), flush=True)
    line = _line(P, args, world, P.GridDims(*GRID), engine_ran, dev_secs, launches, e2e, clk,
                 {"global_grid": [gdims.nx, gdims.ny, gdims.nz],
                  "halo_bytes_per_rank_per_step": halo // max(1, args.steps),
                  "exchange": ("peer stores into the neighbours' halos from the kernel "
                               "(CUDA IPC over NVLink), %d-step passes ordered %s" % (
                                   period, "on the devices by pass counters (no host sync "
                                   "between passes)" if ordered else "by a barrier per pass"))
                              if peer else
                              "torch.distributed %s batch_isend_irecv after every %d-step pass"
                              % (backend, period)})
    if n1:
        line["config"]["n1_same_workload"] = n1
    if e2e_skip:
        line["e2e"]["skipped"] = ("host RAM: %d local ranks x %.0f GB of pinned slab arrays > 70%% "
                                  "of %.0f GB available" % (local_ranks, rank_bytes / 1e9, avail / 1e9))
    dist.destroy_process_group()
    return line if rank == 0 else None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--engine", default="auto",
                    choices=["auto", "split", "fused", "tblock", "tblock-inplace"])
    ap.add_argument("--iters", type=int, default=None)
    ap.add_argument("--device", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-n1-base", action="store_true",
                    help="N>1: skip the one-GPU run of the per-rank workload")
    ap.add_argument("--tile-y", type=int, default=0)
    ap.add_argument("--z-chunk", type=int, default=0)
    ap.add_argument("--schedule", type=int, default=0,
                    help="TBLOCK CTA schedule: 0 auto (rounds, banded tiles), 1 one launch")
    ap.add_argument("--band", type=int, default=0, help="TBLOCK rounds: tile columns per band")
    ap.add_argument("--time-block", type=int, default=0,
                    help="TBLOCK steps per HBM pass: 0 auto, 2, 3")
    ap.add_argument("--config", default=None, choices=sorted(CONFIGS),
                    help="default: configs[2] at N=1, configs[4] (per rank) at N>1")
    ap.add_argument("--check", type=int, default=0,
                    help="multi-rank: also run CHECK steps and compare with the oracle (rank 0)")
    ap.add_argument("--coeff", default="full", choices=["full", "table"],
                    help="coefficient layout; 'table' (material ids, layered configs only) is "
                         "reported separately from the reference-layout roofline")
    args = ap.parse_args()
    global GRID, ITERS, KIND, WORKLOAD
    world, rank, local = dist_env()
    if args.config is None:
        args.config = default_config(world)
    GRID, ITERS, KIND, desc = CONFIGS[args.config]
    if args.iters is None:
        args.iters = ITERS
    WORKLOAD = (desc + " (H then E half-step) per bench step, complex128, fields U[-1,1], "
                + ("per-layer coeffs" if KIND else "coeffs") + " |c|<=0.45, seed 1, zero halo")
    if args.impl == "reference":
        run_reference_arm(args, world, rank)
    else:
        run_native(args, world, rank, local)


if __name__ == "__main__":
    main()
