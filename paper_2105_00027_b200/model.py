"""Ring, K1 and memory models of the B200 ring: SURVEY.md section 8f, row 4.

The reference carries two closed-form models for the Summit-era machine. This
module keeps them and re-parameterises them for one NVSwitch node of B200s:

* ``ringacc.perf`` (perf.py:53-124): per measurement, each rank of a sub-ring
  sends and receives S-1 messages, and the elapsed time is set by the slowest
  link's per-step service time.  :func:`message_counts`, :func:`slow_link`,
  :func:`predict_elapsed` and :func:`model_utilization` restate it with the
  same arguments and results (tests/golden/models.json pins them against the
  reference).  :data:`NVSWITCH_B200` is the B200 link set.  All 8 GPUs of a
  node sit behind NVSwitch: every ring step is an "intra" transfer at the
  measured peer-copy rate, and the NIC only matters for rings that span nodes.
* ``ringacc.memory`` (memory.py:26-115): :func:`make_plan` keeps the
  reference's itemised per-rank plan and break-even lane count.
  :func:`device_plan` adds what this implementation really allocates per GPU:
  the slice, 3 staged payload buffers per lane and walker of a batch
  (engine.RingEngine), and the staged layout's halo.  It answers "how large a
  G4 fits on 8 x 180 GB".

New here, because on B200 the question is whether a ring step hides behind
the slice update:

* :func:`k1_pass_time` models one K1 launch from its three bounds.  These are
  the same per-update byte and instruction counts the bench line reports in
  ``roofline`` / ``onchip``: HBM bytes, bytes through
  the SM shared-memory/L1 data path, and FP instructions.  Each bound is
  divided by the efficiency this kernel reaches on it, calibrated from the
  round-1 bench lines (tests check the model against them).
* :func:`ring_round_time` models one measurement round of the ring engine.
  The own payload is applied first, then S-1 steps.  Each step's transfer
  overlaps the previous K1 pass, so a step costs max(K1, transfer).
  :func:`hide_planes` gives the smallest per-GPU slice that hides the ring.
  :func:`scaling_table` gives whole-job updates/s for 1, 2, 4 and 8 GPUs.

Run ``python -m paper_2105_00027_b200.model`` for the tables of BASELINE
configs 2-4.
"""
from __future__ import annotations

import argparse
import ctypes
import json
from dataclasses import dataclass

from . import _lib
from .errors import ConfigError, ContractViolation

# ---------------------------------------------------------------------------
# reference perf model (perf.py), same arguments and results


@dataclass(frozen=True)
class LinkConfig:
    """Link parameters (transport/sim.py:34-60): bandwidths in bytes/s, latency in s."""

    nic_bandwidth: float = 12.5e9
    intra_bandwidth: float = 25e9
    latency: float = 5e-6
    ranks_per_node: int = 6

    def __post_init__(self):
        if self.nic_bandwidth <= 0 or self.intra_bandwidth <= 0:
            raise ConfigError("link bandwidths must be strictly positive")
        if self.latency <= 0:
            raise ConfigError("link latency must be strictly positive")
        if self.ranks_per_node < 1:
            raise ConfigError("ranks_per_node must be >= 1")


# One DGX-class B200 node: the peer-copy rate over NVLink 5 / NVSwitch
# (B200_PROFILING.md: ~770 GB/s per direction of the 900 GB/s nominal). The
# per-step latency covers a copy-engine launch plus the stream flag write and
# wait of engine.py (assumed, not measured: only one GPU per gpurun call). One
# 400 Gb/s NIC per GPU is used between nodes.
NVSWITCH_B200 = LinkConfig(nic_bandwidth=50e9, intra_bandwidth=770e9, latency=8e-6, ranks_per_node=8)


def message_counts(subring_size: int) -> tuple[int, int, int, int]:
    """(per-rank sends, per-rank receives, total, per link) for one measurement
    of one lane (perf.py:53-58)."""
    if subring_size < 1:
        raise ContractViolation("subring size must be >= 1")
    s = subring_size
    return (s - 1, s - 1, s * (s - 1), s - 1)


def slow_link(subring_size: int, link: LinkConfig, lanes: int = 1) -> tuple[str, int, float]:
    """(link class, per-step message load, bandwidth) of the busiest link under
    block placement (perf.py:87-104).  A pair link carries its pair's k lane
    messages.  A node-boundary NIC carries one egress and one ingress per lane."""
    candidates = []
    if link.ranks_per_node >= 2 and subring_size >= 2:
        candidates.append(("intra", lanes, link.intra_bandwidth))
    if subring_size > link.ranks_per_node:
        candidates.append(("nic", 2 * lanes, link.nic_bandwidth))
    if not candidates:
        return ("intra", lanes, link.intra_bandwidth)
    return max(candidates, key=lambda c: c[1] / c[2])


def predict_elapsed(subring_size: int, n_meas: int, msg_bytes: float, link: LinkConfig,
                    lanes: int = 1) -> float:
    """Transfer-only elapsed time of the ring pattern on the slowest link
    (perf.py:107-116): n_meas * (S-1) * (latency + msg * load / bandwidth)."""
    if subring_size < 1:
        raise ConfigError("subring size must be >= 1")
    if subring_size == 1:
        return 0.0
    _, load, bandwidth = slow_link(subring_size, link, lanes)
    return n_meas * (subring_size - 1) * (link.latency + msg_bytes * load / bandwidth)


def model_utilization(subring_size: int, link: LinkConfig, lanes: int = 1) -> float:
    """Fraction of the slow link's bandwidth one lane stream gets per step (perf.py:119-124)."""
    return 1.0 / slow_link(subring_size, link, lanes)[1]


# ---------------------------------------------------------------------------
# reference memory model (memory.py), same results

BUFFERS_PER_LANE_ORIGINAL = 1
BUFFERS_PER_LANE_DISTRIBUTED = 3
BUFFERS_PER_LANE_ALTERNATE = 2


def slice_bytes(total: int, p: int) -> int:
    """Largest balanced share of ``total`` over p ranks (memory.py:33-37)."""
    if p < 1:
        raise ContractViolation(f"rank count must be >= 1, got {p}")
    return -(-total // p)


def gsigma_total_bytes(mode: str, k: int, matrix_bytes: float) -> float:
    """Per-rank payload buffers: matrix_bytes * 2 spins * buffers * k lanes (memory.py:40-50)."""
    if k < 1:
        raise ContractViolation(f"lane count must be >= 1, got {k}")
    buffers = {"original": BUFFERS_PER_LANE_ORIGINAL, "distributed": BUFFERS_PER_LANE_DISTRIBUTED}.get(mode)
    if buffers is None:
        raise ContractViolation(f"unknown mode {mode!r}")
    return matrix_bytes * 2 * buffers * k


def make_plan(entries: int, entry_bytes: int, matrix_bytes: float, p: int, k: int) -> dict:
    """The reference's itemised per-rank plan (memory.py:91-115), as its to_dict():
    totals are sums of their parts; ``break_even_k`` is the lane count at which
    the distributed algorithm stops saving memory."""
    if entries < 0:
        raise ContractViolation(f"entry count must be >= 0, got {entries}")
    gt_total = entries * entry_bytes
    gt_rank = slice_bytes(gt_total, p)
    orig = gsigma_total_bytes("original", k, matrix_bytes)
    dist = gsigma_total_bytes("distributed", k, matrix_bytes)
    extra_per_k = (BUFFERS_PER_LANE_DISTRIBUTED - BUFFERS_PER_LANE_ORIGINAL) * 2 * matrix_bytes
    saved = gt_total - gt_rank
    return {
        "gt_bytes_total": gt_total, "gt_bytes_per_rank": gt_rank, "gsigma_matrix_bytes": matrix_bytes,
        "p": p, "k": k, "buffers_per_lane": BUFFERS_PER_LANE_DISTRIBUTED,
        "gsigma_bytes_original": orig, "gsigma_bytes_distributed": dist,
        "gsigma_bytes_alternate_2_per_lane": matrix_bytes * 2 * BUFFERS_PER_LANE_ALTERNATE * k,
        "original_total_per_rank": gt_total + orig, "distributed_total_per_rank": gt_rank + dist,
        "break_even_k": saved / extra_per_k if extra_per_k > 0 else float("inf"),
    }


# ---------------------------------------------------------------------------
# B200 device plan

B200_HBM_BYTES = 180e9     # usable HBM3e per GPU (bench --max-g4 measured 189.7 GB free of 191.5 GB)
_DTYPE = {"c128": _lib.G4_C128, "c64": _lib.G4_C64, "mixed": _lib.G4_C128_G64}


def _check_dtype(dtype: str) -> None:
    if dtype not in _DTYPE:
        raise ConfigError(f"dtype must be one of {sorted(_DTYPE)}")


def entry_bytes(dtype: str) -> int:
    """Bytes of one G4 entry (complex128 unless the whole path is complex64)."""
    _check_dtype(dtype)
    return 8 if dtype == "c64" else 16


def payload_entry_bytes(dtype: str) -> int:
    _check_dtype(dtype)
    return 16 if dtype == "c128" else 8


def staged_payload_bytes(n: int, dtype: str) -> int:
    """Bytes of one walker in the staged (halo'd, ring-wire) layout: g4_payload_bytes."""
    _check_dtype(dtype)
    code = _lib.G4_C128 if dtype == "c128" else _lib.G4_C64
    return int(_lib.load().g4_payload_bytes(n, code))


def wire_payload_bytes(n: int, dtype: str) -> int:
    """Bytes of one walker on the ring: the N x N cores of both spins (g4_copy_payload_cores)."""
    return 2 * n * n * payload_entry_bytes(dtype)


def device_plan(n: int, planes_total: int, gpus: int, lanes: int = 1, batch: int = 1,
                dtype: str = "c128", hbm_bytes: float = B200_HBM_BYTES) -> dict:
    """Per-GPU allocation of the ring engine: the G4 slice plus, per channel,
    3 x batch x lanes staged payloads (GEN, R0, R1, engine.py:262).  It also gives
    the largest slice that still fits, and the G4 the whole ring can hold."""
    if min(n, planes_total, gpus, lanes, batch) < 1:
        raise ContractViolation("device_plan arguments must be >= 1")
    plane = n * n * entry_bytes(dtype)
    per_gpu_planes = -(-planes_total // gpus)
    pay = staged_payload_bytes(n, dtype)
    ring = BUFFERS_PER_LANE_DISTRIBUTED * batch * lanes * pay
    slice_b = per_gpu_planes * plane
    max_planes = int((hbm_bytes - ring) // plane) if hbm_bytes > ring else 0
    return {
        "n": n, "dtype": dtype, "gpus": gpus, "planes_per_gpu": per_gpu_planes,
        "slice_bytes": slice_b, "payload_bytes": pay, "ring_buffer_bytes": ring,
        "total_bytes": slice_b + ring, "fits": slice_b + ring <= hbm_bytes,
        "g4_total_bytes": planes_total * plane,
        "max_planes_per_gpu": max_planes, "max_g4_bytes": max_planes * plane * gpus,
        "halo_overhead": pay / (2 * n * n * payload_entry_bytes(dtype)) - 1.0,
    }


# ---------------------------------------------------------------------------
# K1 and ring time models

@dataclass(frozen=True)
class K1Calibration:
    """Measured ceilings and the fraction of each that K1 reaches (round-1
    profiles: profiles/r01_summary.md, tools/microbench.cu)."""

    hbm_gbs: float = 6450.0            # MEASURED_PEAKS.json hbm_gbs (driver-measured copy bandwidth)
    smem_b_per_clk_sm: float = 126.0   # conflict-free LDS.128
    sm_clock_hz: float = 1965e6
    sms: int = 148
    fp64_instr_per_s: float = 17.0e12  # DFMA issue
    fp32_instr_per_s: float = 35.7e12  # FFMA issue
    eff_hbm: float = 0.86              # B = 1: 0.84-0.88 of HBM (r01j; 0.71 in r01c)
    eff_smem: float = 0.78             # exact, N = 512: B = 8 / 16 at 0.72 / 0.88 of the smem data path (r01j)
    eff_fp: float = 0.85
    launch_s: float = 4e-6             # launch + tail of one pass
    # K1 v3 (the persistent TMEM-hand-off kernel): the slice traffic and the
    # math overlap only partly; time = w_hbm * HBM time + w_fp * FP64 issue time
    # at peak, fitted on the round-2 lines (N = 512 B = 8 and 16; checked at
    # N = 1024 and 4608 within 8 %, profiles/r02e_bench*.json)
    v3_w_hbm: float = 0.684
    v3_w_fp: float = 1.123

    @property
    def smem_bytes_per_s(self) -> float:
        return self.smem_b_per_clk_sm * self.sms * self.sm_clock_hz


B200_K1 = K1Calibration()


def k1_geometry(n: int, planes: int, dtype: str, nbatch: int = 8, arith: str | None = None) -> dict:
    """The launch g4_accumulate_staged picks for this shape (g4_k1_config), under
    the given arithmetic mode ("exact" / "fused"), or the library's current one."""
    _check_dtype(dtype)
    lib = _lib.load()
    out = (ctypes.c_int32 * 9)()
    prev = lib.g4_get_arith_mode()
    if arith is not None:
        _lib.check(lib.g4_set_arith_mode(_lib.G4_ARITH_FUSED if arith == "fused" else _lib.G4_ARITH_EXACT))
    try:
        _lib.check(lib.g4_k1_config(n, planes, nbatch, _DTYPE[dtype], out), "k1_config")
    finally:
        _lib.check(lib.g4_set_arith_mode(prev))
    v = list(out)
    return {"variant": v[0], "pp": v[1], "dd": v[2], "q": v[3], "dr": v[4], "stages": v[5],
            "ctas_per_sm": v[6], "warps": v[7], "deferred": bool(v[8])}


def k1_pass_time(n: int, planes: int, batch: int, dtype: str = "c128", arith: str = "exact",
                 cal: K1Calibration = B200_K1) -> dict:
    """Modelled time of one K1 launch (B walkers over a P-plane slice) and its bounds."""
    if min(n, planes, batch) < 1:
        raise ContractViolation("k1_pass_time arguments must be >= 1")
    g = k1_geometry(n, planes, dtype, batch, arith)
    eb, peb = entry_bytes(dtype), payload_entry_bytes(dtype)
    upd = batch * planes * n * n
    hbm_b = 2 * planes * n * n * eb + batch * 2 * n * n * peb
    lds = 2 * peb * (g["pp"] + 2 * g["dd"] - 1) / (g["pp"] * g["dd"])
    width = 32 if peb == 16 else 34
    fill = 2 * peb * width * (g["dr"] + g["q"] + g["dr"] - 1) / (g["q"] * g["dr"] * 32) if g["variant"] >= 2 else 0.0
    smem_b = upd * (lds + fill + (0.0 if g["deferred"] else 2 * eb / batch))
    fp_i = upd * (8 if arith == "fused" else 12)
    fpeak = cal.fp32_instr_per_s if dtype == "c64" else cal.fp64_instr_per_s
    # wave quantisation: the last wave of CTAs leaves SMs idle
    ctas = -(-planes // g["q"]) * -(-n // 32) * -(-n // g["dr"])
    resident = cal.sms * g["ctas_per_sm"]
    util = ctas / (-(-ctas // resident) * resident)
    bounds = {"hbm": hbm_b / (cal.hbm_gbs * 1e9 * cal.eff_hbm),
              "smem": smem_b / (cal.smem_bytes_per_s * cal.eff_smem * util),
              "fp": fp_i / (fpeak * cal.eff_fp * util)}
    if g["variant"] == 3:
        bounds["v3"] = (cal.v3_w_hbm * hbm_b / (cal.hbm_gbs * 1e9) + cal.v3_w_fp * fp_i / fpeak) / util
    elif g["deferred"]:
        # The deferred update's L2 read-modify-write and the payload fills share
        # the L2 <-> SM path and do not overlap: the r01j fused lines (B = 8, 16;
        # N = 512 and 4608) sit within 7 % of the SUM of the two times at peak.
        bounds["hbm+smem"] = hbm_b / (cal.hbm_gbs * 1e9) + smem_b / (cal.smem_bytes_per_s * util)
    bound = max(bounds, key=bounds.get)
    t = bounds[bound] + cal.launch_s
    return {"time_s": t, "bound": bound, "bounds_s": bounds, "updates": upd, "hbm_bytes": hbm_b,
            "updates_per_s": upd / t, "geometry": g, "wave_utilisation": util}


def ring_round_time(gpus: int, batch: int, n: int, planes_total: int, dtype: str = "c128",
                    lanes: int = 1, subring_size: int | None = None, arith: str = "exact",
                    link: LinkConfig = NVSWITCH_B200, cal: K1Calibration = B200_K1) -> dict:
    """One measurement round of the ring engine on ``gpus`` GPUs in sub-rings of S.
    * Each GPU owns planes_total / S planes of its sub-ring's copy.
    * Each lane contributes ``batch`` walkers per round.
    * A step moves batch x lanes staged payloads and runs one K1 pass over them.
    The sub-ring's copies are reduced once at the end of a run, which is not
    part of a round."""
    s = subring_size or gpus
    if gpus % s:
        raise ConfigError("subring size must divide the GPU count")
    p = -(-planes_total // s)
    walkers = batch * lanes
    k1 = k1_pass_time(n, p, walkers, dtype, arith, cal)
    # only the N x N cores cross the link; the receiver rebuilds the halo (HBM read + write)
    msg = walkers * wire_payload_bytes(n, dtype)
    halo_s = walkers * 2 * (staged_payload_bytes(n, dtype) - wire_payload_bytes(n, dtype)) / (cal.hbm_gbs * 1e9)
    k1 = dict(k1, time_s=k1["time_s"] + (halo_s if s > 1 else 0.0))
    _, load, bw = slow_link(s, link, 1)
    xfer = link.latency + msg * load / bw if s > 1 else 0.0
    step = max(k1["time_s"], xfer)
    round_s = k1["time_s"] + (s - 1) * step
    upd = gpus * walkers * p * n * n * s  # every GPU applies all S x walkers payloads of its sub-ring
    return {"gpus": gpus, "subring_size": s, "planes_per_gpu": p, "walkers_per_pass": walkers,
            "k1_s": k1["time_s"], "k1_bound": k1["bound"], "transfer_s": xfer, "message_bytes": msg,
            "round_s": round_s, "hidden": xfer <= k1["time_s"],
            "compute_fraction": s * k1["time_s"] / round_s if round_s > 0 else 1.0,
            "nvlink_bytes_per_round_per_gpu": (s - 1) * msg, "updates_per_s": upd / round_s}


def hide_planes(n: int, batch: int, dtype: str = "c128", lanes: int = 1, arith: str = "exact",
                link: LinkConfig = NVSWITCH_B200, cal: K1Calibration = B200_K1, max_planes: int = 4096) -> int:
    """Smallest per-GPU slice (planes) whose K1 pass hides one ring step
    (0 if none up to ``max_planes``)."""
    msg = batch * lanes * wire_payload_bytes(n, dtype)
    xfer = link.latency + msg / link.intra_bandwidth
    lo, hi = 1, max_planes
    if k1_pass_time(n, hi, batch * lanes, dtype, arith, cal)["time_s"] < xfer:
        return 0
    while lo < hi:
        mid = (lo + hi) // 2
        if k1_pass_time(n, mid, batch * lanes, dtype, arith, cal)["time_s"] >= xfer:
            hi = mid
        else:
            lo = mid + 1
    return lo


def scaling_table(n: int, planes_total: int, batch: int, dtype: str = "c128", lanes: int = 1,
                  gpu_counts=(1, 2, 4, 8), subring_size: int | None = None, arith: str = "exact") -> list[dict]:
    """Predicted weak scaling of the bench's ring workload (each GPU adds ``batch`` walkers per lane)."""
    rows = []
    base = None
    for g in gpu_counts:
        s = min(subring_size or g, g)
        r = ring_round_time(g, batch, n, planes_total, dtype, lanes, s, arith)
        if base is None:
            base = r["updates_per_s"] / g
        r["efficiency"] = r["updates_per_s"] / (g * base)
        rows.append(r)
    return rows


CONFIGS = {
    # name: (n_k, n_w, planes, gpus, subring size, lanes) -- BASELINE.json configs
    "c2": (16, 32, 64, 8, 8, 1),
    "c3": (16, 64, 64, 8, 4, 2),
    "c4": (36, 128, 576, 8, 8, 1),
}


def main(argv=None) -> None:
    ap = argparse.ArgumentParser(description=__doc__.split("\n\n")[0])
    ap.add_argument("--config", default="all", choices=["all", *CONFIGS])
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--json", action="store_true")
    a = ap.parse_args(argv)
    out = {}
    for name in (CONFIGS if a.config == "all" else [a.config]):
        n_k, n_w, planes, gpus, s, lanes = CONFIGS[name]
        n = n_k * n_w
        out[name] = {}
        for dtype in ("c128", "mixed"):
            out[name][dtype] = {
                "scaling": scaling_table(n, planes, a.batch, dtype, lanes, subring_size=s),
                "hide_planes": hide_planes(n, a.batch, dtype, lanes),
                "memory": device_plan(n, planes, s, lanes, a.batch, dtype),
            }
    if a.json:
        print(json.dumps(out, indent=1))
        return
    for name, by_dt in out.items():
        for dtype, d in by_dt.items():
            m = d["memory"]
            print(f"{name} {dtype}: N={m['n']}, {m['planes_per_gpu']} planes/GPU "
                  f"({m['slice_bytes'] / 1e9:.2f} GB + ring {m['ring_buffer_bytes'] / 1e9:.2f} GB), "
                  f"ring hidden from {d['hide_planes']} planes/GPU, "
                  f"max G4 on 8 GPUs {m['max_g4_bytes'] / 1e12:.2f} TB")
            for r in d["scaling"]:
                print(f"   {r['gpus']} GPU(s) S={r['subring_size']}: {r['updates_per_s']:.3e} upd/s, "
                      f"eff {r['efficiency']:.2f}, K1 {r['k1_s'] * 1e6:.0f} us ({r['k1_bound']}) vs "
                      f"step {r['transfer_s'] * 1e6:.0f} us -> {'hidden' if r['hidden'] else 'ring-bound'}")


if __name__ == "__main__":
    main()
