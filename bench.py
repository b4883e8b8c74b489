#!/usr/bin/env python
"""Benchmark of the G4 ring-accumulation hot path (BASELINE.json metric:
"G4 updates/sec & HBM GB/s per GPU at 1/2/4/8 B200; max G4 size; vs CPU ref").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--batch B] [--dtype c128|c64]
    torchrun --nproc-per-node N bench.py --gpus N ...          (N > 1: the ring)
    python bench.py --impl reference ...                      (CPU reference arm)

Workload (BASELINE config 2): Nc=16 x 32 frequencies -> N = 512 combined
indices; exchange planes K3 in [0, 64) (16 momenta x 4 frequencies under
K = w*n_k + k); complex128; synthetic payloads from the reference's
counter-based generator (run on the device).  One "step" = one measurement
round: every rank contributes B walkers, the walkers travel the S-rank ring
(S = N GPUs), and every rank applies all S*B walkers to its 64/S planes.
At N=1 a step is one K1 pass of B walkers over the 64-plane slice (268 MB,
larger than L2, so no flush is needed between steps).

value  = G4 updates/s of the whole job (payloads resident in HBM).
e2e    = the same through the reference-facing C ABI (g4_accumulate) with
         payloads in pinned HOST memory in reference layout: H2D copy +
         stage (K2) + update (K1) + D2H of a probe row of the slice per step.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIGS = {
    # name: (n_k, n_w, planes, description)
    "c1": (4, 8, 1, "Nc=4 (2x2), 8 freqs, K3={0}"),
    "c2": (16, 32, 64, "Nc=16 (4x4), 32 freqs, 16 k x 4 w exchange planes"),
    "c3": (16, 64, 64, "Nc=16, 64 freqs, 64 exchange planes"),
    "c4": (36, 128, 576, "Nc=36 (6x6), 128 freqs, 36 k x 16 w exchange planes"),
}
# a single GPU cannot hold config 4's 196 GB G4: at N=1 it runs the per-GPU share of
# the 8-GPU ring (576 / 8 = 72 planes, 24.5 GB) -- stated in the JSON config
SINGLE_GPU_PLANES = {"c4": 72}


def workload(args):
    """(n_k, n_w, planes, description) of the run: BASELINE config `--config`;
    config 4 on one GPU is its per-GPU share of the 8-GPU ring."""
    n_k, n_w, planes, desc = CONFIGS[args.config]
    if args.gpus == 1 and args.config in SINGLE_GPU_PLANES:
        planes = SINGLE_GPU_PLANES[args.config]
        desc += f" -- per-GPU share on one GPU: {planes} planes"
    if args.gpus == 1 and args.planes:
        planes = args.planes
    return n_k, n_w, planes, desc


def ring_shape(args, n_ranks):
    """Sub-ring size S and lanes of an N > 1 run (config 3: 2 sub-rings of 4, 2 lanes)."""
    S = args.subring_size or (min(4, n_ranks) if args.config == "c3" else n_ranks)
    lanes = args.lanes or (2 if args.config == "c3" else 1)
    return S, lanes


def workload_config(args, n_ranks):
    """The JSON `config` object -- identical in both arms (ours and --impl
    reference) for the same flags and N, so the driver can match them."""
    n_k, n_w, planes, desc = workload(args)
    n = n_k * n_w
    eb = 8 if args.dtype == "c64" else 16
    if n_ranks == 1:
        return {"workload": f"{args.config}: {desc}", "n": n, "planes": planes, "walkers_per_pass": args.batch,
                "subring_size": 1, "lanes": 1,
                "l2": ("slice larger than L2 (no flush needed)" if planes * n * n * eb > 126e6
                       else "slice fits L2 (L2-resident caveat)")}
    from oracle import oracle as O
    S, lanes = ring_shape(args, n_ranks)
    p_local = max(hi - lo for lo, hi in O.partition(planes, S))
    return {"workload": f"{args.config}: {desc}", "n": n, "planes": planes, "planes_per_gpu": p_local,
            "walkers_per_rank_per_step": args.batch, "subring_size": S, "lanes": lanes,
            "lane_pipelines": "merged per direction" if (lanes == 1 or args.merged_lanes) else "one per lane",
            "parallelism": f"{n_ranks // S} sub-ring(s) of {S}"}


def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            d = json.loads(p.read_text())
            return float(d["hbm_gbs"]), "measured"
        except Exception:
            pass
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled DURING the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 9:
                self.rows.append(parts)

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[5 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ---------------------------------------------------------------------------
# CPU side (reference arm and cpu_baseline): the numpy port of accumulate_g4
# (oracle/oracle.py, "kind": "port") in one process per host core, each on a
# disjoint K3 range (make_partition), same payloads -- BASELINE.md section 2.

def _cpu_worker(conn, n, lo, hi, walkers, seed):
    import numpy as np
    from oracle import oracle as O
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    gs = [O.gsigma(seed, 0, w, 0, n, "float") for w in range(walkers)]
    g4 = np.zeros((hi - lo, n, n), np.complex128)
    while True:
        msg = conn.recv()
        if msg is None:
            break
        t0 = time.perf_counter()
        for up, down in gs[:msg]:
            O.accumulate_np(g4, lo, hi, up, down)
        conn.send(time.perf_counter() - t0)


class CpuPool:
    def __init__(self, n, planes, walkers, cores, seed=0):
        import multiprocessing as mp
        from oracle import oracle as O
        ctx = mp.get_context("fork")
        self.cores = max(1, min(cores, planes))
        self.ranges = O.partition(planes, self.cores)
        self.conns, self.procs = [], []
        for lo, hi in self.ranges:
            a, b = ctx.Pipe()
            p = ctx.Process(target=_cpu_worker, args=(b, n, lo, hi, walkers, seed), daemon=True)
            p.start()
            self.conns.append(a)
            self.procs.append(p)

    def step(self, walkers):
        t0 = time.perf_counter()
        for c in self.conns:
            c.send(walkers)
        worker_t = [c.recv() for c in self.conns]
        return time.perf_counter() - t0, max(worker_t)

    def close(self):
        for c in self.conns:
            c.send(None)
        for p in self.procs:
            p.join(timeout=10)


def cpu_throughput(n, planes, walkers, steps, warmup, cores):
    pool = CpuPool(n, planes, walkers, cores)
    try:
        for _ in range(warmup):
            pool.step(walkers)
        times = [pool.step(walkers)[0] for _ in range(steps)]
    finally:
        pool.close()
    upd = planes * n * n * walkers
    return upd / statistics.mean(times), statistics.mean(times), pool.cores


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_reference(args):
    """--impl reference: the reference algorithm on the host cores (rank 0 only)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import oracle as O
    n_k, n_w, planes, desc = workload(args)
    n = n_k * n_w
    cores = O.cpu_count()
    n_ranks = int(os.environ.get("WORLD_SIZE", "1"))
    # a bounded sample of the workload per step (B walkers over all planes); updates/s is a
    # per-update rate, so the sample is the same at every N (the CPU does not scale with N)
    walkers = args.batch
    rate, step_s, used = cpu_throughput(n, planes, walkers, args.steps, args.warmup, cores)
    line = {
        "metric": "G4 updates/s", "value": rate, "unit": "updates/s", "impl": "reference",
        "n_gpus": args.gpus, "device": "cpu (all host cores; the same work at every N)", "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_s * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "c128",
        "data": "synthetic (reference generator, float mode, seed 0)",
        "config": workload_config(args, n_ranks),
        "cpu_baseline": {"value": rate, "unit": "updates/s", "cores": used, "kind": "port",
                         "sample": f"{walkers} walkers x {planes} planes x N^2={n * n} per step, "
                                   f"numpy port of accumulate_g4 in {used} processes on disjoint "
                                   f"K3 ranges; host {cpu_model()}"},
        "e2e": {"value": rate, "unit": "updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------

def run_gpu(args):
    import torch
    import torch.distributed as dist

    from paper_2105_00027_b200 import _lib
    from paper_2105_00027_b200 import tensor as T

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    # one GPU per rank; ranks beyond the visible GPUs share them round-robin
    # (how the multi-rank path is exercised on a single-GPU box)
    dev = torch.device("cuda", local % max(torch.cuda.device_count(), 1))
    torch.cuda.set_device(dev)
    if world > 1:
        # control plane only (rendezvous, IPC-handle exchange, barriers); the ring's
        # data path is peer memory + copy engines + stream flags (engine.py)
        dist.init_process_group("gloo")
        return run_ring(args)

    lib = _lib.load()
    _lib.check(lib.g4_set_arith_mode(_lib.G4_ARITH_FUSED if args.arith == "fused" else _lib.G4_ARITH_EXACT))
    n_k, n_w, planes, desc = workload(args)
    sp = T.CombinedIndexSpace(n_k, n_w)
    n = sp.size
    dtype = torch.complex64 if args.dtype == "c64" else torch.complex128    # G4 slice
    pdtype = torch.complex128 if args.dtype == "c128" else torch.complex64  # payloads
    eb = 16 if dtype == torch.complex128 else 8
    peb = 16 if pdtype == torch.complex128 else 8
    B = args.batch
    sl = T.GtSlice.zeros(sp, 0, planes, device=dev, dtype=dtype)
    pools = [[T.GSigma.empty(sp, device=dev, dtype=pdtype) for _ in range(B)] for _ in range(2)]
    for i, pool in enumerate(pools):
        T.fill_gsigmas(pool, 0, [T.Origin(0, 0, w, i, 0) for w in range(B)], "float")
    stream = torch.cuda.current_stream(dev)

    def step(i):
        T.accumulate_g4_batch(sl, pools[i % 2])

    # W warm-up steps, continued to >= 0.5 s of GPU work so that a cold GPU's
    # clocks and the L2 reach steady state before timing
    t_w = time.perf_counter()
    i = 0
    while i < args.warmup or time.perf_counter() - t_w < 0.5:
        step(i)
        i += 1
        if i % 8 == 0:
            torch.cuda.synchronize()
    torch.cuda.synchronize()
    # The timed region holds only K1 launches, back to back on `stream`: their
    # mean duration is the region's event time / steps (gaps included, so
    # conservative).  Per-launch event pairs would serialise consecutive K1
    # launches (+5 us per pass, tools/loop_ab.py).
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        time.sleep(0.3)  # let the sampler start
        torch.cuda.synchronize()
        t_start.record(stream)
        for i in range(args.steps):
            step(i)
        t_end.record(stream)
        torch.cuda.synchronize()
    total_ms = t_start.elapsed_time(t_end)
    launched_geom = int(lib.g4_last_k1_geometry())
    k_ms = [total_ms / args.steps]
    upd_step = B * planes * n * n
    value = upd_step * args.steps / (total_ms * 1e-3)
    peak, peak_kind = measured_peaks()
    alg_bytes = 2 * planes * n * n * eb + B * 2 * n * n * peb
    achieved = alg_bytes / (statistics.mean(k_ms) * 1e-3) / 1e9

    # -- e2e: reference-layout payloads in pinned host memory through g4_accumulate --
    e2e = None if args.skip_extras else run_e2e(args, lib, T, sp, planes, dtype, eb, dev)
    # -- the timed kernel's output, checked after timing (sampled planes vs the C oracle) --
    parity = parity_check(T, sl, pools[0], planes, n, dtype, args.arith)

    line = {
        "metric": "G4 updates/s", "value": value, "unit": "updates/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": args.dtype, "arith": args.arith,
        "parity": ("bitwise vs the reference" if args.arith == "exact"
                   else "within 1e-10 relative (north_star; tests 1e-12), integer payloads bitwise"),
        "data": "synthetic (reference counter-based generator on device, float mode, seed 0)",
        "config": workload_config(args, 1),
        "hbm_gbs": achieved,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": k1_traffic(lib, n, planes, B, args.dtype, args.arith),
                     "peak_source": peak_kind, "kernel": "k_accumulate",
                     "bytes_per_launch": alg_bytes},
        "onchip": onchip_bounds(lib, n, planes, args.dtype, args.arith, B, upd_step / (statistics.mean(k_ms) * 1e-3)),
        "launched_k1_geometry": launched_geom,  # g4_last_k1_geometry() after the timed region (40/43 = K1 v3)
        "clocks": clk.summary(),
        "e2e": e2e,
        "parity_check": parity,
        "gpu_launches": args.steps,
        "g4_bytes": sl.nbytes,
    }
    if not args.skip_extras:
        line["batch_sweep"] = batch_sweep(T, sl, sp, pdtype, dev, planes, n, eb, peb, peak, B)
        line["other_arith"] = other_arith_point(lib, _lib, T, sl, sp, pdtype, dev, planes, n, eb, peb, peak, B,
                                                args.arith)
        line["max_g4"] = max_g4_capacity(dev, walkers=B)
    if args.config == "c2" and not args.planes and not args.skip_extras:
        del sl, pools
        torch.cuda.empty_cache()
        line["config_points"] = config_points(T, dev, dtype, pdtype, eb, peb, peak)
    if not args.no_cpu_baseline:
        from oracle import oracle as O
        cores = O.cpu_count()
        rate, step_s, used = cpu_throughput(n, planes, B, max(2, args.cpu_steps), 1, cores)
        line["cpu_baseline"] = {
            "value": rate, "unit": "updates/s", "cores": used, "kind": "port",
            "sample": f"{max(2, args.cpu_steps)} steps of {B} walkers x {planes} planes x N^2={n * n}, "
                      f"numpy port of accumulate_g4 in {used} processes on disjoint K3 ranges; "
                      f"host {cpu_model()}"}
        # also one core (8 planes of the same shape; the rate is per update)
        rate1, _, _ = cpu_throughput(n, min(8, planes), B, 2, 1, 1)
        line["cpu_baseline"]["one_core"] = {"value": rate1, "unit": "updates/s", "cores": 1,
                                            "sample": f"2 steps of {B} walkers x {min(8, planes)} planes"}
    print(json.dumps(line), flush=True)


def parity_check(T, sl, walkers, planes, n, dtype, arith, sample=(0, None, -1)):
    """One more pass of the timed launch configuration, from a zeroed slice
    with the first walker pool, then sampled planes (first, middle, last)
    against the C oracle (test infrastructure, used here only as the checker,
    after the timed region).  Bitwise expected in exact mode; fused mode is
    judged against 1e-12 relative (complex64 slices: 1e-5)."""
    import numpy as np
    import torch
    from oracle import oracle as O
    sl.data.zero_()
    T.accumulate_g4_batch(sl, walkers)
    torch.cuda.synchronize()
    qs = sorted({q if q is not None and q >= 0 else (planes // 2 if q is None else planes + q) for q in sample})
    host = [(g.up.contiguous().cpu().numpy().astype(np.complex128),
             g.down.contiguous().cpu().numpy().astype(np.complex128)) for g in walkers]
    worst, bitwise = 0.0, True
    for q in qs:
        got = sl.data[q].cpu().numpy().astype(np.complex128)
        ref = np.zeros((1, n, n), np.complex128)
        for up, down in host:
            O.accumulate(ref, q, q + 1, up, down)
        if dtype == torch.complex64:
            ref = ref.astype(np.complex64).astype(np.complex128)
        bitwise &= bool(np.array_equal(got, ref[0]))
        worst = max(worst, float(np.abs(got - ref[0]).max() / max(np.abs(ref).max(), 1e-300)))
    tol = 1e-5 if dtype == torch.complex64 else (0.0 if arith == "exact" else 1e-12)
    return {"planes": qs, "walkers": len(walkers), "max_rel_err": worst, "bitwise": bitwise, "tol": tol,
            "ok": bool(worst <= tol), "checker": "oracle/g4_oracle.c (C restatement of tensor.py:233-251)"}


def k1_traffic(lib, n, planes, B, dtype, arith):
    """DRAM bytes per K1 launch from the committed ncu capture of this exact
    launch configuration (profiles/k1_traffic.json), else None."""
    import ctypes
    cfg = (ctypes.c_int32 * 9)()
    lib.g4_k1_config(n, planes, B, {"c128": 0, "c64": 1, "mixed": 2}[dtype], cfg)
    v = list(cfg)
    key = f"v{v[0]}/{v[1]}x{v[2]}/{v[3]}x{v[4]}/{v[5]} n={n} planes={planes} B={B} {dtype} {arith}"
    try:
        d = json.loads((ROOT / "profiles" / "k1_traffic.json").read_text()).get(key)
    except (OSError, ValueError):
        return None
    return None if d is None else d["dram_read_bytes"] + d["dram_write_bytes"]


# On-chip ceilings of K1 (calibrated with tools/microbench.cu, profiles/r01_microbench.txt):
# conflict-free LDS.128 126 B/clk/SM, DFMA 17.0 T instr/s, FFMA 35.7 T instr/s.
SMEM_B_PER_CLK_SM = 126.0
FP64_INSTR_PEAK = 17.0e12
FP32_INSTR_PEAK = 35.7e12


def batch_sweep(T, sl, sp, pdtype, dev, planes, n, eb, peb, peak, B_main, batches=(1, 16), steps=6):
    """Secondary points of the same K1 on the same slice (not the headline),
    timed like the headline: two walker pools alternate, so no step re-reads
    the previous step's L2-resident payloads.  B = 1 is the HBM-bound end,
    B = 16 the on-chip-bound end."""
    import torch
    out = {}
    for B in batches:
        if B == B_main:
            continue
        pools = [[T.GSigma.empty(sp, device=dev, dtype=pdtype) for _ in range(B)] for _ in range(2)]
        for i, pool in enumerate(pools):
            T.fill_gsigmas(pool, 1, [T.Origin(0, 0, w, 90 + i, 0) for w in range(B)], "float")
        for i in range(4):
            T.accumulate_g4_batch(sl, pools[i % 2])
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(dev)
        a.record()
        for i in range(steps):
            T.accumulate_g4_batch(sl, pools[i % 2])
        b.record()
        torch.cuda.synchronize(dev)
        s = a.elapsed_time(b) * 1e-3 / steps
        byt = 2 * planes * n * n * eb + B * 2 * n * n * peb
        out[str(B)] = {"updates_per_s": B * planes * n * n / s, "hbm_frac": byt / s / 1e9 / peak,
                       "us_per_pass": s * 1e6}
    return out


# Per-GPU K1 work of the other BASELINE configs, timed on this GPU like the headline
# (secondary points; the 8-GPU runs themselves need an 8-GPU node):
# (name, n_k, n_w, planes, walkers per pass, description)
CONFIG_POINTS = [
    ("c3_share", 16, 64, 16, 16, "config 3 per-GPU K1 pass: N=1024, 64 planes over sub-rings of 4 -> 16 planes, "
                                 "2 lanes x 8 walkers in one pass"),
    ("c3_full", 16, 64, 64, 8, "config 3 index space on one GPU: N=1024, all 64 planes, 8 walkers"),
    ("c4_share", 36, 128, 72, 8, "config 4 per-GPU share of the 8-GPU ring: N=4608, 72 planes (24.5 GB), "
                                 "8 walkers"),
]


def config_points(T, dev, dtype, pdtype, eb, peb, peak, steps=5):
    """K1 throughput and HBM fraction for each CONFIG_POINTS entry: its own
    slice and two walker pools (alternating), >= 3 warm-up passes, event-timed
    back-to-back passes."""
    import torch
    out = {}
    for name, n_k, n_w, planes, B, desc in CONFIG_POINTS:
        sp = T.CombinedIndexSpace(n_k, n_w)
        n = sp.size
        sl = T.GtSlice.zeros(sp, 0, planes, device=dev, dtype=dtype)
        pools = [[T.GSigma.empty(sp, device=dev, dtype=pdtype) for _ in range(B)] for _ in range(2)]
        for i, pool in enumerate(pools):
            T.fill_gsigmas(pool, 2, [T.Origin(0, 0, w, 50 + i, 0) for w in range(B)], "float")
        for i in range(3):
            T.accumulate_g4_batch(sl, pools[i % 2])
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(dev)
        a.record()
        for i in range(steps):
            T.accumulate_g4_batch(sl, pools[i % 2])
        b.record()
        torch.cuda.synchronize(dev)
        t = a.elapsed_time(b) * 1e-3 / steps
        byt = 2 * planes * n * n * eb + B * 2 * n * n * peb
        out[name] = {"workload": desc, "n": n, "planes": planes, "walkers_per_pass": B,
                     "updates_per_s": B * planes * n * n / t, "hbm_frac": byt / t / 1e9 / peak,
                     "us_per_pass": t * 1e6, "g4_bytes": sl.nbytes,
                     "l2": "slice larger than L2" if sl.nbytes > 126e6 else "slice fits L2 (L2-resident caveat)"}
        del sl, pools
        torch.cuda.empty_cache()
    return out


def other_arith_point(lib, _lib, T, sl, sp, pdtype, dev, planes, n, eb, peb, peak, B, arith, steps=10):
    """The same workload in the other arithmetic mode, as a secondary point.
    exact: the reference's op order, bitwise equal to it.  fused: FMA chains
    plus (B >= 4) the deferred L2-reduction update of the slice; within the
    north_star 1e-10 relative (tests check 1e-12; integer payloads bitwise)."""
    other = "exact" if arith == "fused" else "fused"
    _lib.check(lib.g4_set_arith_mode(_lib.G4_ARITH_FUSED if other == "fused" else _lib.G4_ARITH_EXACT))
    try:
        out = batch_sweep(T, sl, sp, pdtype, dev, planes, n, eb, peb, peak, 0, batches=(B,), steps=steps)[str(B)]
    finally:
        _lib.check(lib.g4_set_arith_mode(_lib.G4_ARITH_FUSED if arith == "fused" else _lib.G4_ARITH_EXACT))
    out.update(arith=other, walkers_per_pass=B,
               parity="bitwise vs the reference" if other == "exact" else "1e-10 relative (north_star); tests 1e-12")
    return out


def onchip_bounds(lib, n, planes, dtype, arith, B, upd_per_s):
    """Per-update traffic through each SM's shared-memory/L1 data path and FP
    instruction count of the K1 launch actually used (g4_k1_config), with the
    fraction of each measured ceiling the kernel reaches.  At B >= 4 these,
    not HBM, bound K1."""
    import ctypes
    import torch
    code = {"c128": 0, "c64": 1, "mixed": 2}[dtype]
    cfg = (ctypes.c_int32 * 9)()
    lib.g4_k1_config(n, planes, B, code, cfg)
    variant, pp, dd, q, dr, nst, ctas, warps, deferred = list(cfg)
    eb = 8 if dtype == "c64" else 16          # G4 entry
    peb = 16 if dtype == "c128" else 8        # payload entry
    lds = 2 * peb * (pp + 2 * dd - 1) / (pp * dd)            # operand loads per update
    width = 32 if peb == 16 else 34
    fill = 2 * peb * width * (dr + q + dr - 1) / (q * dr * 32) if variant >= 2 else 0.0  # TMA writes
    g4 = 0.0 if deferred else 2 * eb / B                     # G4 block in and out through L1 (deferred: L2 reduction)
    path = lds + fill + g4
    props = torch.cuda.get_device_properties(torch.cuda.current_device())
    clock_hz = 1965e6
    smem_peak = SMEM_B_PER_CLK_SM * props.multi_processor_count * clock_hz
    instr = (8 if arith == "fused" else 12)
    fpeak = FP32_INSTR_PEAK if dtype == "c64" else FP64_INSTR_PEAK
    return {
        "k1": {"variant": variant, "thread_block": [pp, dd], "cta_tile": [q, dr], "stages": nst,
               "ctas_per_sm": ctas, "warps_per_cta": warps, "deferred_update": bool(deferred)},
        "smem_path_bytes_per_update": {"operand_lds": lds, "tma_fill": fill, "g4_via_l1": g4, "total": path},
        "smem_path_achieved_TBps": path * upd_per_s / 1e12,
        "smem_path_peak_TBps": smem_peak / 1e12,
        "smem_frac": path * upd_per_s / smem_peak,
        "fp_instr_per_update": instr, "fp_pipe": "fp32" if dtype == "c64" else "fp64",
        "fp_achieved_Tinstr": instr * upd_per_s / 1e12, "fp_peak_Tinstr": fpeak / 1e12,
        "fp_frac": instr * upd_per_s / fpeak,
        "peak_source": "tools/microbench.cu (profiles/r01_microbench.txt) at 1965 MHz",
    }


def max_g4_capacity(dev, n=4608, walkers=8, margin=6e9):
    """Largest complex128 G4 slice (planes of N x N) that fits next to `walkers`
    staged payloads on this GPU; and the 8-GPU total (BASELINE config 4 scale)."""
    import torch
    from paper_2105_00027_b200 import tensor as T
    free, total = torch.cuda.mem_get_info(dev)
    payload = 2 * int(__import__("numpy").prod(T.staged_shape(n)[1:])) * 16
    plane = n * n * 16
    planes = int((free - walkers * payload - margin) // plane)
    return {"n": n, "planes_per_gpu": planes, "bytes_per_gpu": planes * plane,
            "bytes_8gpu": 8 * planes * plane, "gpu_free_bytes": free, "gpu_total_bytes": total,
            "config4_bytes": 576 * plane}


def run_max_g4(args):
    """--max-g4: allocate the largest N=4608 complex128 slice that fits this GPU,
    apply one device-generated walker in one K1 pass, verify the first and last
    planes against the C oracle (test infrastructure, host)."""
    import numpy as np
    import torch
    from oracle import oracle as O
    from paper_2105_00027_b200 import tensor as T
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    cap = max_g4_capacity(dev, walkers=1)
    sp = T.CombinedIndexSpace(36, 128)
    n = sp.size
    planes = cap["planes_per_gpu"]
    sl = T.GtSlice.zeros(sp, 0, planes, device=dev)
    g = T.generate_gsigma(7, T.Origin(0, 0, 0, 0, 0), sp, "float", device=dev)
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    T.accumulate_g4(sl, g)
    t1.record()
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1)
    up, down = O.gsigma(7, 0, 0, 0, n, "float")
    checks = {}
    for k3 in (0, planes - 1):
        ref = np.zeros((1, n, n), np.complex128)
        O.accumulate(ref, k3, k3 + 1, up, down)
        got = sl.data[k3].cpu().numpy()
        checks[k3] = float(np.abs(got - ref[0]).max() / np.abs(ref).max())
    line = {"metric": "max G4 per GPU", "value": sl.nbytes, "unit": "bytes", "planes": planes, "n": n,
            "dtype": "c128", "pass_ms": ms, "pass_gbs": 2 * sl.nbytes / (ms * 1e-3) / 1e9,
            "verified_planes_max_rel_err": checks, "ok": all(v < 1e-10 for v in checks.values()),
            "capacity": cap}
    print(json.dumps(line), flush=True)


def run_e2e(args, lib, T, sp, planes, dtype, eb, dev):
    import torch
    n = sp.size
    B = args.batch
    code = 2 if args.dtype == "mixed" else _dtype_code(dtype)  # G4_C128_G64 for mixed
    sl = T.GtSlice.zeros(sp, 0, planes, device=dev, dtype=dtype)
    host = []
    for i in range(2):
        ups, downs = [], []
        for w in range(B):
            u, d = T.generate_reference_layout(0, T.Origin(0, 0, w, i, 0), sp, "float", device=dev,
                                               dtype=dtype)
            ups.append(u.cpu().pin_memory())
            downs.append(d.cpu().pin_memory())
        host.append((ups, downs))
    dev_bufs = [([torch.empty((n, n), dtype=dtype, device=dev) for _ in range(B)],
                 [torch.empty((n, n), dtype=dtype, device=dev) for _ in range(B)]) for _ in range(2)]
    ws_bytes = lib.g4_accumulate_workspace_bytes(n, B, code)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
    probe = torch.empty(n, dtype=dtype).pin_memory()
    comp = torch.cuda.current_stream(dev)
    copy = torch.cuda.Stream(dev)
    from paper_2105_00027_b200 import _lib
    ready = [torch.cuda.Event() for _ in range(2)]
    done = [torch.cuda.Event() for _ in range(2)]

    def h2d(i):
        j = i % 2
        with torch.cuda.stream(copy):
            copy.wait_event(done[j])
            for w in range(B):
                dev_bufs[j][0][w].copy_(host[j][0][w], non_blocking=True)
                dev_bufs[j][1][w].copy_(host[j][1][w], non_blocking=True)
            ready[j].record(copy)

    def compute(i):
        j = i % 2
        comp.wait_event(ready[j])
        _lib.check(lib.g4_accumulate(
            sl.data.data_ptr(), 0, planes, n, _lib.ptr_array([t.data_ptr() for t in dev_bufs[j][0]]),
            _lib.ptr_array([t.data_ptr() for t in dev_bufs[j][1]]), B, code, 0, ws.data_ptr(),
            ws_bytes, comp.cuda_stream), "g4_accumulate")
        done[j].record(comp)
        probe.copy_(sl.data[0, 0], non_blocking=True)

    for j in range(2):
        done[j].record(comp)
    steps, warm = args.steps, args.warmup
    h2d(0)
    for i in range(warm):
        if i + 1 < warm:
            h2d(i + 1)
        compute(i)
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # every timed step's H2D is issued inside the timed region (the first one
    # after t0, then each one double-buffered under the previous step's compute)
    t0.record(comp)
    copy.wait_event(t0)
    h2d(warm)
    for i in range(warm, warm + steps):
        if i + 1 < warm + steps:
            h2d(i + 1)
        compute(i)
    t1.record(comp)
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1)
    h2d_bytes = B * 2 * n * n * eb
    return {"value": B * planes * n * n * steps / (ms * 1e-3), "unit": "updates/s",
            "h2d_bytes_per_step": h2d_bytes, "d2h_bytes_per_step": n * eb,
            "h2d_gbs_achieved": h2d_bytes * steps / (ms * 1e-3) / 1e9,
            "h2d_peak_gbs": pinned_h2d_peak(dev),
            "path": "g4_accumulate (C ABI, reference layout) from pinned host buffers; "
                    "H2D double-buffered on a copy stream; D2H probe row per step"}


def pinned_h2d_peak(dev, nbytes=256 << 20, reps=5):
    """Measured pinned host -> device copy bandwidth (GB/s): the ceiling of
    the e2e leg, whose per-step H2D of the walkers' reference-layout G's is
    its bound."""
    import torch
    src = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    dst = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize(dev)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        dst.copy_(src, non_blocking=True)
    b.record()
    torch.cuda.synchronize(dev)
    return nbytes * reps / (a.elapsed_time(b) * 1e-3) / 1e9


def _dtype_code(dtype):
    import torch
    return 0 if dtype == torch.complex128 else 1


def run_ring(args):
    """N > 1: the full ring (BASELINE config 2 shape): S = N ranks, each owning
    planes/N exchange planes; every rank contributes B walkers per round; a
    step = one round (own K1 pass + S-1 ring steps, transfers overlapped).
    Payloads are resident in HBM (generated once before timing)."""
    import torch
    import torch.distributed as dist

    from paper_2105_00027_b200 import _lib
    from paper_2105_00027_b200 import engine as E
    from paper_2105_00027_b200 import tensor as T

    lib = _lib.load()
    _lib.check(lib.g4_set_arith_mode(_lib.G4_ARITH_FUSED if args.arith == "fused" else _lib.G4_ARITH_EXACT))
    world = E.Control()
    rank, n_ranks = world.rank, world.size
    n_k, n_w, planes, desc = workload(args)
    B = args.batch
    # BASELINE config 3 is 8 GPUs as 2 sub-rings of 4 with 2 walker streams (lanes) per GPU
    S, lanes = ring_shape(args, n_ranks)
    # several lanes: each its own ring pipeline (comm stream, flags, buffers) -- config 3's
    # "walker streams feeding independent ring pipelines"; --merged-lanes shares one channel
    cfg = E.ExperimentConfig(n_k=n_k, n_w=n_w, world_size=n_ranks, subring_size=S, lanes=lanes,
                             measurements=B, seed=0, value_mode="float", planes=planes, batch=B,
                             dtype={"mixed": "c128g64"}.get(args.dtype, args.dtype), gather=False,
                             instrument=False, timeout_s=120.0,
                             lane_rings=lanes > 1 and not args.merged_lanes)
    E.validate_config(cfg)
    dev = E.device_for_rank(rank)
    torch.cuda.set_device(dev)
    sub = E.build_subrings(world, S)
    eng = E.RingEngine(cfg, sub, rank, dev)
    n = eng.space.size
    eb = 8 if args.dtype == "c64" else 16  # G4 slice entry (mixed: complex128 slice)
    # resident payloads: generate GEN once (K3), untimed
    eng.enqueue_round()
    eng.wait_idle(120.0)
    for i in range(args.warmup):
        eng.enqueue_round(regenerate=False)
    eng.wait_idle(120.0)
    world.barrier()
    torch.cuda.synchronize(dev)
    eng.kernel_events = []
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    nvl = NvlinkCounters(dev.index)
    with ClockSampler(dev.index) as clk:
        time.sleep(0.3)
        world.barrier()
        torch.cuda.synchronize(dev)
        nvl.start()
        t0.record(eng.compute)
        h0 = time.perf_counter()
        for i in range(args.steps):
            eng.enqueue_round(regenerate=False)
        host_ms = (time.perf_counter() - h0) * 1e3 / args.steps
        t1.record(eng.compute)
        eng.wait_idle(300.0)
        torch.cuda.synchronize(dev)
        nvl.stop()
        world.barrier()
    ms_local = t0.elapsed_time(t1) / args.steps
    props = torch.cuda.get_device_properties(dev)
    stats = world.allgather({"ms": ms_local, "k_ms": eng.k1_mean_ms(), "clk": clk.summary(),
                             "lo": eng.lo, "hi": eng.hi, "host_ms": host_ms, "nvlink": nvl.result(args.steps),
                             "device": {"index": dev.index, "pci_bus_id": getattr(props, "pci_bus_id", None),
                                        "uuid": str(getattr(props, "uuid", ""))}})
    e2e = run_ring_e2e(args, eng, world, dev)
    eng_native = eng.native
    eng_wire_cores = eng.wire_cores
    eng.close()
    if rank != 0:
        return
    ms = max(x["ms"] for x in stats)
    kms = max(x["k_ms"] for x in stats)
    # every rank applies the S x B x lanes payloads of its sub-ring to planes / S planes
    upd_step = n_ranks * B * lanes * planes * n * n
    value = upd_step / (ms * 1e-3)
    p_local = max(x["hi"] - x["lo"] for x in stats)
    peak, peak_kind = measured_peaks()
    # one K1 launch applies B x lanes walkers to the rank's p_local planes
    peb = 16 if args.dtype == "c128" else 8
    alg_bytes = 2 * p_local * n * n * eb + B * lanes * 2 * n * n * peb
    achieved = alg_bytes / (kms * 1e-3) / 1e9
    ring_bytes = (S - 1) * B * lanes * eng.wire_bytes
    line = {
        "metric": "G4 updates/s", "value": value, "unit": "updates/s", "n_gpus": n_ranks,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": args.dtype, "arith": args.arith,
        "data": "synthetic (reference counter-based generator on device, float mode, seed 0; resident)",
        "config": workload_config(args, n_ranks),
        "devices": {"visible": torch.cuda.device_count(), "ranks": n_ranks,
                    "ranks_per_device": -(-n_ranks // max(torch.cuda.device_count(), 1)),
                    "rank_devices": [x["device"] for x in stats],
                    "comm": "torch.distributed gloo control plane (no NCCL communicator: payloads move by "
                            "copy engine over CUDA IPC peer memory, flags by cuStreamWrite/WaitValue64)"},
        "per_gpu_updates_per_s": value / n_ranks,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak,
                     "traffic": k1_traffic(lib, n, p_local, B * lanes, args.dtype, args.arith),
                     "peak_source": peak_kind, "kernel": "k_accumulate*", "bytes_per_launch": alg_bytes,
                     "walkers_per_launch": B * lanes, "planes_per_launch": p_local},
        "nvlink": {"bytes_per_step_per_gpu": ring_bytes,
                   "wire": "payload cores" if eng_wire_cores else "staged payloads",
                   "achieved_gbs": ring_bytes / (ms * 1e-3) / 1e9, "peak_gbs": 770.0,
                   "peak_source": "B200_PROFILING.md measured peer copy",
                   "achieved_note": "wire bytes / step time (computed); measured counters per rank below",
                   "measured_per_rank": [x["nvlink"] for x in stats]},
        "clocks": stats[0]["clk"],
        "clocks_per_rank": [x["clk"] for x in stats],
        "e2e": e2e,
        "host": {"enqueue_ms_per_step": max(x["host_ms"] for x in stats),
                 "native_rounds": eng_native,
                 "note": "host time to issue one round (one C call with the native round program)"},
        "model": ring_model_line(n, planes, n_ranks, B, args.dtype, S, lanes),
        "gpu_launches": args.steps * S,  # K1 launches per rank per step = S (own + S-1 received)
    }
    print(json.dumps(line), flush=True)


class NvlinkCounters:
    """NVLink data bytes this GPU sent and received during the timed region,
    from NVML's throughput counters (nvmlDeviceGetFieldValues,
    NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX/RX, KiB, summed over links), read
    before and after.  On a GPU without active NVLinks (or a driver that does
    not expose the fields) the result says so instead of a number."""

    TX, RX = 138, 139  # NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX / _RX

    def __init__(self, gpu_index: int):
        self.err = None
        self.h = None
        self.a = self.b = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(gpu_index)
        except Exception as exc:  # NVML absent
            self.err = f"nvml unavailable: {exc}"

    def _read(self):
        vals = self.nvml.nvmlDeviceGetFieldValues(self.h, [self.TX, self.RX])
        out = []
        for v in vals:
            if v.nvmlReturn != 0:
                raise RuntimeError(f"field {v.fieldId}: nvml return {v.nvmlReturn}")
            out.append(int(v.value.ullVal) * 1024)
        return out

    def start(self):
        if self.h is not None:
            try:
                self.a = self._read()
            except Exception as exc:
                self.err = str(exc)

    def stop(self):
        if self.h is not None and self.a is not None:
            try:
                self.b = self._read()
            except Exception as exc:
                self.err = str(exc)

    def result(self, steps: int) -> dict:
        if self.a is None or self.b is None:
            return {"source": "nvml", "unavailable": self.err or "not read"}
        tx, rx = self.b[0] - self.a[0], self.b[1] - self.a[1]
        return {"source": "nvml NVLINK_THROUGHPUT_DATA_TX/RX", "tx_bytes_per_step": tx / steps,
                "rx_bytes_per_step": rx / steps}


def ring_model_line(n, planes, gpus, batch, dtype, subring_size, lanes):
    """The NVLink-5 ring model's prediction for this run (paper_2105_00027_b200.model)."""
    from paper_2105_00027_b200 import model as M
    r = M.ring_round_time(gpus, batch, n, planes, dtype, lanes, subring_size)
    return {"round_ms": r["round_s"] * 1e3, "k1_ms": r["k1_s"] * 1e3, "step_transfer_ms": r["transfer_s"] * 1e3,
            "ring_hidden": r["hidden"], "updates_per_s": r["updates_per_s"],
            "hide_from_planes_per_gpu": M.hide_planes(n, batch, dtype),
            "link": "NVSwitch B200 (770 GB/s per direction, 8 us per step; model.NVSWITCH_B200)"}


def run_ring_e2e(args, eng, world, dev):
    """Ring e2e: each rank's walkers arrive in pinned host memory (reference
    layout); per step H2D (double-buffered on a copy stream, overlapping the
    previous round) + stage (K2) + round + D2H of a probe row."""
    import torch
    B = args.batch * eng.cfg.lanes  # walkers staged per rank per round (all lanes)
    n = eng.space.size
    dtype = eng.dtype
    ups = [torch.randn(n, n, dtype=dtype).pin_memory() for _ in range(B)]
    downs = [torch.randn(n, n, dtype=dtype).pin_memory() for _ in range(B)]
    dev_bufs = [([torch.empty((n, n), dtype=dtype, device=dev) for _ in range(B)],
                 [torch.empty((n, n), dtype=dtype, device=dev) for _ in range(B)]) for _ in range(2)]
    probe = torch.empty(n, dtype=dtype).pin_memory()
    copy = torch.cuda.Stream(dev)
    ready = [torch.cuda.Event() for _ in range(2)]
    done = [torch.cuda.Event() for _ in range(2)]
    for j in range(2):
        done[j].record(eng.compute)
    eng.kernel_events = None

    def h2d(i):
        j = i % 2
        with torch.cuda.stream(copy):
            copy.wait_event(done[j])
            for w in range(B):
                dev_bufs[j][0][w].copy_(ups[w], non_blocking=True)
                dev_bufs[j][1][w].copy_(downs[w], non_blocking=True)
            ready[j].record(copy)

    def step(i):
        j = i % 2
        with torch.cuda.stream(eng.compute):
            eng.compute.wait_event(ready[j])
            eng.stage_gen(dev_bufs[j][0], dev_bufs[j][1])
            done[j].record(eng.compute)
            eng.enqueue_round(regenerate=False)
            probe.copy_(eng.slice.data[0, 0], non_blocking=True)

    h2d(0)
    for i in range(2):
        h2d(i + 1)
        step(i)
    eng.wait_idle(120.0)
    world.barrier()
    torch.cuda.synchronize(dev)
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(eng.compute)
    copy.wait_event(t0)
    h2d(2)
    for i in range(args.steps):
        if i + 1 < args.steps:
            h2d(3 + i)
        step(2 + i)
    t1.record(eng.compute)
    eng.wait_idle(300.0)
    torch.cuda.synchronize(dev)
    ms = max(world.allgather(t0.elapsed_time(t1) / args.steps))
    eb = 16 if dtype == torch.complex128 else 8
    return {"value": world.size * B * eng.cfg.num_planes * n * n / (ms * 1e-3),  # B includes lanes
            "unit": "updates/s", "h2d_bytes_per_step": B * 2 * n * n * eb, "d2h_bytes_per_step": n * eb,
            "path": "pinned host walkers -> H2D (copy stream, double-buffered) -> g4_prepare_g (K2) "
                    "-> ring round; D2H probe row"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--batch", type=int, default=8, help="walkers per K1 pass (per rank)")
    ap.add_argument("--dtype", default="c128", choices=["c128", "c64", "mixed"],
                    help="mixed: complex128 G4 slice with complex64 payloads")
    ap.add_argument("--arith", default="fused", choices=["exact", "fused"],
                    help="exact: reference op order (bitwise); fused: FMA-chained (within 1e-10)")
    ap.add_argument("--cpu-steps", type=int, default=3)
    ap.add_argument("--planes", type=int, default=0, help="override the exchange-plane count (N=1)")
    ap.add_argument("--max-g4", action="store_true", help="allocate + update + verify the largest N=4608 slice")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--skip-extras", action="store_true",
                    help="lab runs: headline + parity check only (no e2e, sweeps, other configs)")
    ap.add_argument("--subring-size", type=int, default=0, help="ring size S for N > 1 (default N; c3: 4)")
    ap.add_argument("--lanes", type=int, default=0, help="walker streams per GPU for N > 1 (default 1; c3: 2)")
    ap.add_argument("--merged-lanes", action="store_true",
                    help="N > 1: lanes sharing a direction share one ring channel (default: a pipeline per lane)")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    if args.max_g4:
        return run_max_g4(args)
    return run_gpu(args)


if __name__ == "__main__":
    main()
