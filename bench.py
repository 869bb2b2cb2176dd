#!/usr/bin/env python3
"""Benchmark of the B200 Fast DCT+ apply path (the driver's contract).

Headline workload: BASELINE.json configs[4] (C5) — the largest config by work
and the one the north star shards over 1/2/4/8 B200s: path graph n = 8192
plus rho u u^T, rho = 0.1, u_i = gaussian()/sqrt(n) from
Rng(mix_seed(2409, 8192, 50)); forward DCT+ (DctPlusPlan::forward,
fast_transform.hpp:163-195 — the reference's near-pole guard sends it to the
dense X^T s, :199-209) of 2048 fp64 N(0,1) signals drawn with the reference's
Rng (signal.hpp:18-55) from mix_seed(2409, 8192, 5).  The metric spans every
config (n = 64..8192, fp64/fp32); C5 carries the headline because it is the
only config the north star shards across GPUs and the one with the most work
per step.  A step = one forward DCT+ of the whole batch; metric = transformed
(output) samples per second, whole job.

Every other BASELINE config is measured in the same run and reported under
`configs` in the same JSON line: C1, C2, C3 forward and inverse in fp64 and
fp32, C4 (progressive, 16 sets), C5 — each with its dominant-kernel and step
rooflines, an end-to-end number through the public host-buffer API and the
reference's own CPU path on the host cores beside it.

Arms:
  default            this repo's sm_100a kernels through the C ABI.
  --impl reference   the reference's own CPU implementation (oracle/_ref: the
                     unmodified headers compiled here) on all host threads,
                     same metric / config, a bounded sample per step.  This
                     arm never imports the product package: inputs come from
                     the reference's own Rng (ref_rng_fill).

Multi-GPU (torchrun, one process per GPU): strong scaling — the configured
batch is split into contiguous row slices (shard_rows), one plan per device,
no data-path collective and no NCCL (signals are independent); a gloo group
provides the barriers and the max over ranks of the CUDA-event time.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

MEASURED = ROOT / "MEASURED_PEAKS.json"
PEAKS_FILE = ROOT / "profiles" / "peaks_fp64.json"
L2_BYTES = 126 * 2**20
SEED = 2409
METRIC = "DCT+ transformed samples/sec"
UNIT = "samples/s"

# BASELINE.json configs (0-based vertices there, the reference's 1-based
# RankOneUpdate here; kind 0 self_loop, 1 edge_delta, 2 general direction).
# dist: 0 gaussian, 2 AR(r) rows, 3 2u-1, 4 2-D separable AR(r) rows.
_WS = tuple((0, 0.05 + k * (1.95 / 15.0), 1, 0) for k in range(16))
CONFIGS = {
    "C1": dict(cid=1, n=64, batch=4096, dist=0, r=0.0, updates=((0, 0.5, 1, 0),), dtype="f64", op="forward",
               name="C1 n=64 self_loop(1,0.5) forward fp64 batch 4096"),
    "C2": dict(cid=2, n=256, batch=65536, dist=2, r=0.95, updates=((1, -0.7, 128, 129),), dtype="f64",
               op="forward", name="C2 n=256 edge_delta(128,129,-0.7) forward fp64 batch 65536"),
    "C3_fwd_f64": dict(cid=3, n=1024, batch=16384, dist=3, r=0.0, updates=((1, 1.0, 1, 1024),), dtype="f64",
                       op="forward", name="C3 n=1024 edge_delta(1,1024,1.0) forward fp64 batch 16384"),
    "C3_inv_f64": dict(cid=3, n=1024, batch=16384, dist=3, r=0.0, updates=((1, 1.0, 1, 1024),), dtype="f64",
                       op="inverse", name="C3 n=1024 edge_delta(1,1024,1.0) inverse fp64 batch 16384"),
    "C3_fwd_f32": dict(cid=3, n=1024, batch=16384, dist=3, r=0.0, updates=((1, 1.0, 1, 1024),), dtype="f32",
                       op="forward", name="C3 n=1024 edge_delta(1,1024,1.0) forward fp32 batch 16384"),
    "C3_inv_f32": dict(cid=3, n=1024, batch=16384, dist=3, r=0.0, updates=((1, 1.0, 1, 1024),), dtype="f32",
                       op="inverse", name="C3 n=1024 edge_delta(1,1024,1.0) inverse fp32 batch 16384"),
    "C4": dict(cid=4, n=128, batch=65536, dist=4, r=0.9, updates=_WS, dtype="f32", op="forward_all",
               name="C4 n=128 K=16 self_loop(1,w_k) progressive fp32 batch 65536 (16 sets)"),
    "C5": dict(cid=5, n=8192, batch=2048, dist=0, r=0.0, updates=((2, 0.1, 0, 0),), dtype="f64", op="forward",
               name="C5 n=8192 general u~N(0,1/n) rho=0.1 forward fp64 batch 2048"),
    # not BASELINE configs: SURVEY 8(f) rows, `--config X6|X7|X8` only
    "X6": dict(cid=6, n=1024, batch=16384, dist=2, r=0.95, updates=((0, 1.5, 1, 0), (1, -0.5, 1, 1024),
                                                                   (1, 0.25, 300, 700)), dtype="f64",
               op="chain", name="X6 n=1024 rank-3 chain forward fp64 batch 16384"),
    "X7": dict(cid=7, n=1024, batch=16384, dist=0, r=0.0, updates=((0, 0.5, 1, 0),), dtype="f64", op="forward",
               name="X7 n=1024 self_loop(1,0.5) forward fp64 batch 16384 (NFST route)"),
    "X8": dict(cid=8, n=2048, batch=8192, dist=0, r=0.0, updates=((0, 5.0, 1, 0),), dtype="f64", op="forward",
               name="X8 n=2048 self_loop(1,5.0) forward fp64 batch 8192 (NFST route)"),
}
HEADLINE = "C5"
ALL_BASELINE = ("C1", "C2", "C3_fwd_f64", "C3_inv_f64", "C3_fwd_f32", "C3_inv_f32", "C4", "C5")


def out_sets(cfg) -> int:
    """Coefficient sets counted per signal (C4: the 16 member sets; the shared
    DCT set 0 is written too but not counted, SURVEY.md 8 decision 3)."""
    return 16 if cfg["op"] == "forward_all" else 1


def config_dict(cfg) -> dict:
    """The `config` object of the JSON line — identical in both arms."""
    return {"workload": cfg["name"], "n": cfg["n"], "batch": cfg["batch"], "precision": cfg["dtype"],
            "op": cfg["op"], "output_sets": out_sets(cfg)}


def mix_seed(seed: int, size: int, kind: int) -> int:
    """bench.hpp:89-95 (the same constants as the reference)."""
    x = (seed * 0x9E3779B97F4A7C15 + size * 0x100000001B3 + kind + 1) & (2**64 - 1)
    x ^= x >> 33
    x = (x * 0xFF51AFD7ED558CCD) & (2**64 - 1)
    x ^= x >> 33
    return x


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default=HEADLINE, help="headline workload key (C1..C5, C3_inv_f64, ..., X6-X8)")
    ap.add_argument("--no-configs", action="store_true", help="skip the per-config sub-measurements")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--sustain-s", type=float, default=3.0, help="untimed load held after the headline timing")
    return ap.parse_args()


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))


def shard_rows(batch: int, rank: int, world: int):
    base, extra = divmod(batch, world)
    return rank * base + min(rank, extra), base + (1 if rank < extra else 0)


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


# ----------------------------------------------------------------- reference (CPU)

class RefWorkload:
    """The reference's own objects for a config (oracle/_ref: the unmodified
    headers): DctPlusPlan / PrunedEnsemblePlan (c_p = n, thr = DBL_MAX) /
    compose_rank_k; inputs from the reference's Rng (ref_rng_fill)."""

    _cache = {}

    def __init__(self, cfg):
        from oracle import checkers as O

        self.cfg, self.ref = cfg, O.Reference()
        n = cfg["n"]
        ups = []
        for (k, rho, i, j) in cfg["updates"]:
            v = None
            if k == 2:  # config 5's direction, drawn with the reference's Rng
                v = tuple(float(x) for x in self.ref.fill(mix_seed(SEED, n, 50), 0, n, 1)[0] / math.sqrt(n))
            ups.append(O.Update(k, rho, i, j, v))
        key = (n, tuple(cfg["updates"]), cfg["op"] == "forward_all", cfg["op"] == "chain")
        if key not in RefWorkload._cache:
            if cfg["op"] == "chain":
                obj = self.ref.chain(n, ups)
            elif cfg["op"] == "forward_all":
                obj = self.ref.ensemble(n, ups, n, float(np.finfo(np.float64).max))
            else:
                obj = self.ref.plan(n, ups[0])
            RefWorkload._cache[key] = obj
        self.obj = RefWorkload._cache[key]

    def signals(self, rows: int) -> np.ndarray:
        c = self.cfg
        return self.ref.fill(mix_seed(SEED, c["n"], c["cid"]), c["dist"], c["n"], rows, c["r"])

    def runner(self, rows: int, threads: int):
        s = self.signals(rows)
        op = self.cfg["op"]
        if op == "inverse":
            p = self.obj.forward(s, threads=threads)
            return lambda: self.obj.inverse(p, threads=threads)
        if op == "forward_all":
            return lambda: self.obj.forward_all(s, threads=threads)
        return lambda: self.obj.forward(s, threads=threads)


def reference_rate(cfg, threads: int, warmup: int, steps: int, target_s: float):
    """The reference's CPU path on `threads` host threads (one shared plan,
    one workspace per std::thread, contiguous slices: proj/README.md:82-87),
    each step a bounded sample of the workload sized to ~target_s seconds.
    Returns (samples/s, rows per step, per-step seconds)."""
    w = RefWorkload(cfg)
    probe = min(cfg["batch"], max(16, 4 * threads))
    run = w.runner(probe, threads)
    t = time.perf_counter()
    run()
    per = (time.perf_counter() - t) / probe
    rows = int(min(cfg["batch"], max(probe, target_s / max(per, 1e-9))))
    run = w.runner(rows, threads)
    for _ in range(warmup):
        run()
    times = []
    for _ in range(steps):
        t = time.perf_counter()
        run()
        times.append(time.perf_counter() - t)
    value = rows * cfg["n"] * out_sets(cfg) * steps / sum(times)
    return value, rows, times


def cpu_baseline(cfg, warmup: int = 1, steps: int = 3, target_s: float = 1.5) -> dict:
    threads = host_cores()
    try:
        value, rows, _ = reference_rate(cfg, threads, warmup, steps, target_s)
    except Exception as e:  # reference not built on this box
        return {"value": None, "unit": UNIT, "cores": 0, "kind": "reference", "sample": f"unavailable: {e}"}
    return {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
            "sample": f"{rows} of {cfg['batch']} signals per step, {warmup} warm-up + {steps} timed passes, "
                      f"reference {api_name(cfg)} (oracle/_ref, FFTW stand-in) on {threads} threads of {cpu_model()}"}


def api_name(cfg) -> str:
    return {"forward": "DctPlusPlan::forward", "inverse": "DctPlusPlan::inverse",
            "forward_all": "PrunedEnsemblePlan::forward_all", "chain": "chain_forward"}[cfg["op"]]


def run_reference_arm(args, rank: int):
    if rank != 0:
        return
    cfg = CONFIGS[args.config]
    threads = host_cores()
    target = max(0.5, 100.0 / max(1, args.steps + args.warmup))
    value, rows, times = reference_rate(cfg, threads, args.warmup, args.steps, target)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(times) / len(times),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": cfg["dtype"],
        "data": "synthetic: seeded reference Rng (mt19937_64 + Box-Muller) signals of the BASELINE config",
        "config": config_dict(cfg),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                         "sample": f"{rows} of {cfg['batch']} signals per step, reference {api_name(cfg)} "
                                   f"(oracle/_ref, FFTW stand-in) on {threads} threads of {cpu_model()}"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------- clocks

class ClockSampler:
    """nvidia-smi-equivalent sampling (NVML) while it is active."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, index: int):
        self.samples, self.reasons, self.power = [], set(), []
        self.max_mhz = None
        self._stop = threading.Event()
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nvml = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception as e:  # pragma: no cover
            self.nvml, self.err = None, str(e)
        self.t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nvml.nvmlDeviceGetClockInfo(self.h, self.nvml.NVML_CLOCK_SM))
                self.power.append(self.nvml.nvmlDeviceGetPowerUsage(self.h) / 1000.0)
                mask = self.nvml.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if mask & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.nvml:
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nvml:
            self.t.join()

    def report(self):
        if not self.nvml:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples),
                "power_w_max": max(self.power) if self.power else None}


# -------------------------------------------------------------------- GPU arm

def peaks():
    meas = json.loads(MEASURED.read_text()) if MEASURED.exists() else {}
    own = json.loads(PEAKS_FILE.read_text()) if PEAKS_FILE.exists() else {}
    return meas, own


def algorithmic(cfg, plan) -> dict:
    """SURVEY.md 8d, per signal: bytes = elem * n * (1 + K_out); flops =
    2.5 n log2 n (DCT-II) + 2 * n_kept * n_active * K (the direct Cauchy
    stage).  The chain is one dense product (2 n^2, no DCT)."""
    n = cfg["n"]
    elem = 4 if cfg["dtype"] == "f32" else 8
    k = out_sets(cfg)
    if cfg["op"] == "chain":
        return {"bytes": elem * n * 2, "flops_cauchy": 2.0 * n * n, "flops_dct": 0.0, "out_samples": n}
    if cfg["op"] == "forward_all":
        cauchy = sum(2 * m.n_kept * m.n_active for m in (plan.member(r) for r in range(1, 17)))
    else:
        cauchy = 2 * plan.n_kept * plan.n_active
    return {"bytes": elem * n * (1 + k), "flops_cauchy": float(cauchy), "flops_dct": 2.5 * n * math.log2(n),
            "out_samples": n * k}


def kernel_roofline(cfg, alg, rows, top, t_ms, ms_per_step, ozaki_products):
    """Roofline of the dominant kernel: algorithmic work per launch / its
    average launch time, against the measured peak of the unit it runs on."""
    meas, own = peaks()
    hbm_peak = meas.get("hbm_gbs") or 6650.0
    hbm_src = "MEASURED_PEAKS.json hbm_gbs" if meas.get("hbm_gbs") else "B200_PROFILING.md fallback 6650 GB/s"
    nbytes = alg["bytes"] * rows
    f32 = cfg["dtype"] == "f32"
    hbm_ach = nbytes / (t_ms * 1e-3) / 1e9
    out = {"kernel": top, "launch_ms": t_ms, "kernel_share_of_step": t_ms / ms_per_step,
           "algorithmic_bytes_per_launch": nbytes, "hbm_achieved_gbs": hbm_ach, "hbm_frac": hbm_ach / hbm_peak,
           "traffic": None}
    if "bf16x3" in top:
        # fp32 product on the tcgen05 tensor cores with the bf16x3 split: three
        # bf16 MMAs per algorithmic one (tc_bf16x3.cu)
        flops = alg["flops_cauchy"] * rows
        bf = meas.get("bf16_tflops")
        peak = bf / 3.0 if bf else None
        ach = flops / (t_ms * 1e-3) / 1e12
        t_flop = flops / (peak * 1e12) if peak else 0.0
        t_hbm = nbytes / (hbm_peak * 1e9)
        if t_hbm >= t_flop:
            out.update({"bound": "hbm", "unit": "GB/s", "achieved": hbm_ach, "peak": hbm_peak,
                        "frac": hbm_ach / hbm_peak, "peak_source": hbm_src})
        else:
            out.update({"bound": "tensor", "unit": "TFLOP/s", "achieved": ach, "peak": peak,
                        "frac": ach / peak if peak else None,
                        "peak_source": "MEASURED_PEAKS.json bf16_tflops / 3 (bf16x3 passes)"})
        out["algorithmic_flops_per_launch"] = flops
        out["t_roof_ms"] = max(t_flop, t_hbm) * 1e3
        return out
    if top.endswith("_i8"):
        # fp64 product on the int8 tensor cores: the kernel's algorithm is
        # P = S(S+1)/2 int8 GEMMs of the same shape (ozaki.cu); peak = the
        # measured tcgen05 kind::i8 rate (tools/tc_peak.cu)
        # the NFST route's materialised n x n operator: 2 n^2 per signal
        alg_flops = 2.0 * cfg["n"] * cfg["n"] if top.startswith("nfst_dense") else alg["flops_cauchy"]
        ops = ozaki_products * alg_flops * rows
        peak = own.get("tcgen05_i8_tops")
        ach = ops / (t_ms * 1e-3) / 1e12
        fp64_eq = alg_flops * rows / (t_ms * 1e-3) / 1e12
        dmma = max(own.get("dmma_m8n8k4_tflops") or 0, own.get("dmma_m16n8k16_tflops") or 0) or None
        out.update({"bound": "tensor", "unit": "TOPS (int8)", "achieved": ach, "peak": peak,
                    "frac": ach / peak if peak else None,
                    "peak_source": "profiles/peaks_fp64.json tcgen05_i8_tops (tools/tc_peak.cu, measured, "
                                   "128x256x32 kind::i8 from shared memory)",
                    "algorithmic_int8_ops_per_launch": ops, "int8_products": ozaki_products,
                    "fp64_equivalent_tflops": fp64_eq,
                    "fp64_equivalent_vs_dmma_peak": fp64_eq / dmma if dmma else None})
        return out
    product = any(k in top for k in ("cauchy", "fold_w", "dense", "chain", "progressive_sgemm", "progressive_tc32"))
    if "fused" in top:
        flops = (alg["flops_cauchy"] + alg["flops_dct"]) * rows
    elif product:
        flops = alg["flops_cauchy"] * rows
    else:
        flops = 0.0
    if f32 and "tc32" in top:
        tf = own.get("tcgen05_tf32_tflops")
        peak, bound = (tf / 3.0 if tf else None), "tensor"
        src = "profiles/peaks_fp64.json tcgen05_tf32_tflops (tools/tc_peak.cu, measured) / 3 (3xTF32 passes)"
    elif f32:
        peak = max(own.get("fp32_fma_tflops") or 0.0, own.get("fp32_ffma2_tflops") or 0.0) or None
        bound, src = "fp32-fma", "profiles/peaks_fp64.json max(fp32_fma_tflops, fp32_ffma2_tflops) (tools/peaks.cu)"
    else:
        peak = max(own.get("dmma_m8n8k4_tflops") or 0.0, own.get("dmma_m16n8k16_tflops") or 0.0) or None
        bound, src = "tensor", "profiles/peaks_fp64.json max DMMA m8n8k4 / m16n8k16 (tools/peaks.cu, measured)"
    ach = flops / (t_ms * 1e-3) / 1e12
    t_flop = flops / (peak * 1e12) if peak and flops else 0.0
    t_hbm = nbytes / (hbm_peak * 1e9)
    if t_hbm >= t_flop:
        out.update({"bound": "hbm", "unit": "GB/s", "achieved": hbm_ach, "peak": hbm_peak, "frac": hbm_ach / hbm_peak,
                    "peak_source": hbm_src})
    else:
        out.update({"bound": bound, "unit": "TFLOP/s", "achieved": ach, "peak": peak,
                    "frac": ach / peak if peak else None, "peak_source": src,
                    "algorithmic_flops_per_launch": flops})
    out["t_roof_ms"] = max(t_flop, t_hbm) * 1e3
    return out


class GpuArm:
    def __init__(self, args, rank, local, world):
        import torch

        import paper_2409_08970_b200 as P

        self.args, self.rank, self.local, self.world = args, rank, local, world
        self.torch, self.P = torch, P
        torch.cuda.set_device(local)
        self.dev = torch.device("cuda", local)
        if world > 1:
            import torch.distributed as dist

            dist.init_process_group("gloo")  # barriers + max over ranks only: no data-path collective
        self.flush_buf = None
        self.plans = {}

    def barrier(self):
        if self.world > 1:
            self.torch.distributed.barrier()
        self.torch.cuda.synchronize(self.dev)

    def max_over_ranks(self, v: float) -> float:
        if self.world == 1:
            return v
        t = self.torch.tensor([float(v)], dtype=self.torch.float64)
        self.torch.distributed.all_reduce(t, op=self.torch.distributed.ReduceOp.MAX)
        return float(t.item())

    def flush_l2(self):
        if self.flush_buf is None:
            self.flush_buf = self.torch.empty(2 * L2_BYTES // 4, dtype=self.torch.float32, device=self.dev)
        self.flush_buf.fill_(1.0)

    def plan(self, cfg):
        from paper_2409_08970_b200.configs import WORKLOADS, make_plan

        key = cfg["cid"]
        if key not in self.plans:
            t = time.perf_counter()
            self.plans[key] = (make_plan(WORKLOADS[key], device=self.local), time.perf_counter() - t)
        return self.plans[key]

    def measure(self, key, headline=False):
        torch, P, args = self.torch, self.P, self.args
        cfg = CONFIGS[key]
        plan, setup_s = self.plan(cfg)
        n, batch = cfg["n"], cfg["batch"]
        start, rows = shard_rows(batch, self.rank, self.world)
        dtype = torch.float32 if cfg["dtype"] == "f32" else torch.float64
        host = P.fill_signals(P.mix_seed(SEED, n, cfg["cid"]), cfg["dist"], n, batch, cfg["r"])[start:start + rows]
        x = torch.as_tensor(host, device=self.dev).to(dtype)
        op = cfg["op"]
        sets = 17 if op == "forward_all" else 1
        y = torch.empty((rows, sets, n) if op == "forward_all" else (rows, n), dtype=dtype, device=self.dev)
        if op == "inverse":
            x = plan.forward(x)  # the coefficients the inverse takes
            host = x.cpu().numpy()
        if op == "forward_all":
            step = lambda: plan.forward_all_batch(x, sync=False, out=y)  # noqa: E731
        elif op == "inverse":
            step = lambda: plan.inverse(x, sync=False, out=y)  # noqa: E731
        else:
            step = lambda: plan.forward(x, sync=False, out=y)  # noqa: E731
        check = (lambda: plan.sync_check()) if hasattr(plan, "sync_check") else (lambda: None)
        elem = 4 if dtype == torch.float32 else 8
        in_bytes = rows * n * elem
        big = in_bytes > L2_BYTES  # inputs larger than L2: no flush needed between steps
        stream = torch.cuda.current_stream(self.dev)
        steps, warm = args.steps, max(3, args.warmup)
        for _ in range(warm):
            step()
        if op != "forward_all":
            check()
        self.barrier()

        clocks = ClockSampler(self.local) if headline else None
        if clocks:
            clocks.__enter__()
        if big:
            # exactly `steps` back-to-back steps bracketed by barrier + sync,
            # CUDA events on the launching stream
            self.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(steps):
                step()
            e1.record(stream)
            self.barrier()
            ms = e0.elapsed_time(e1)
            l2 = f"inputs {in_bytes / 2**20:.0f} MiB per rank per step > 126 MB L2: no flush"
        else:
            # inputs fit in L2: the K steps rotate over R copies of the input
            # and output (R x (in + out) > 2 x L2, so every step reads its
            # input from DRAM), captured in one CUDA graph so the host-side
            # launch path is not inside the timed region either
            out_bytes = y.numel() * y.element_size()
            reps = max(2, -(-2 * L2_BYTES // (in_bytes + out_bytes)))
            xs = [x.clone() for _ in range(reps)]
            ys = [torch.empty_like(y) for _ in range(reps)]

            def step_i(i):
                xi, yi = xs[i % reps], ys[i % reps]
                if op == "forward_all":
                    plan.forward_all_batch(xi, sync=False, out=yi)
                elif op == "inverse":
                    plan.inverse(xi, sync=False, out=yi)
                else:
                    plan.forward(xi, sync=False, out=yi)

            gs = torch.cuda.Stream(self.dev)
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.stream(gs):
                for i in range(reps):  # first-use allocations outside the capture
                    step_i(i)
                torch.cuda.synchronize(self.dev)
                with torch.cuda.graph(graph, stream=gs):
                    for i in range(steps):
                        step_i(i)
            graph.replay()
            self.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            graph.replay()
            e1.record(stream)
            self.barrier()
            ms = e0.elapsed_time(e1)
            if op != "forward_all":
                check()
            l2 = (f"inputs {in_bytes / 2**20:.1f} MiB per rank fit in L2: the {steps} timed steps rotate over {reps} "
                  f"input/output copies ({reps * (in_bytes + out_bytes) / 2**20:.0f} MiB > 2 x 126 MB L2), "
                  f"captured in one CUDA graph")
        # per-kernel times (the library's CUDA events around every launch): a
        # separate untimed pass of the same steps right after the timed one
        # (same clocks; the same L2 flush between steps for small inputs)
        P.profile_reset()
        P.profile_enable(True)
        for _ in range(steps):
            if not big:
                self.flush_l2()
            step()
        torch.cuda.synchronize(self.dev)
        P.profile_enable(False)
        prof = P.profile_summary()
        if not big:
            # per-launch events include the launch latency of these short
            # kernels; scale the kernels' shares to the graph-timed step
            tot = sum(v[1] for v in prof.values()) / steps
            prof = {k: (v[0], v[1] * (ms / steps) / tot) for k, v in prof.items()}
        sustain = None
        if clocks:
            # untimed sustained load so the clocks (ours and the driver's
            # sampler) are seen under load
            t_end = time.perf_counter() + args.sustain_s
            k = 0
            while time.perf_counter() < t_end:
                for _ in range(8):
                    step()
                torch.cuda.synchronize(self.dev)
                k += 8
            sustain = {"seconds": args.sustain_s, "steps": k}
            clocks.__exit__()
        ms = self.max_over_ranks(ms)
        ms_per_step = ms / steps
        alg = algorithmic(cfg, plan)
        value = batch * alg["out_samples"] * steps / (ms * 1e-3)

        per_launch = {k: v[1] / max(v[0], 1) for k, v in prof.items()}
        launches = {k: v[0] / steps for k, v in prof.items()}
        top = max(prof, key=lambda k: prof[k][1])
        S = ctypes_ozaki_slices(n)
        if top == "nfst_dense_inv_i8":
            S = 6  # the NFST adjoint's materialised operator takes 6 slices (capi.cpp nfst_dense_slices)
        roof = kernel_roofline(cfg, alg, rows, top, per_launch[top], ms_per_step, S * (S + 1) // 2)
        meas, _ = peaks()
        hbm_peak = meas.get("hbm_gbs") or 6650.0
        step_bytes = alg["bytes"] * batch
        roof["step_hbm_gbs"] = step_bytes / (ms_per_step * 1e-3) / 1e9
        roof["step_hbm_frac"] = roof["step_hbm_gbs"] / hbm_peak
        tfile = ROOT / "profiles" / "traffic.json"
        tmap = json.loads(tfile.read_text()) if tfile.exists() else {}
        rec = tmap.get(key)
        if rec and rec.get("kernel") == top:
            roof["traffic"] = rec["dram_bytes_per_launch"]
            roof["traffic_source"] = rec["source"]

        e2e = self.e2e(cfg, plan, host, rows, dtype, sets, alg)
        res = {"value": value, "unit": UNIT, "ms_per_step": ms_per_step, "steps": steps, "l2": l2,
               "roofline": roof, "e2e": e2e, "setup_s": setup_s,
               "kernels": {k: {"launches_per_step": launches[k], "ms_per_launch": per_launch[k]} for k in prof},
               "gpu_launches": int(round(sum(launches.values()) * steps))}
        if clocks:
            res["clocks"] = clocks.report()
            res["sustained_load"] = sustain
        return res

    def e2e(self, cfg, plan, host, rows, dtype, sets, alg):
        """The public host-buffer entry (what DctPlusPlan.forward(numpy) calls)
        on pinned buffers: per step the H2D of the inputs, the transform and
        the D2H of the coefficients, synchronous; wall clock, max over ranks."""
        import ctypes as C

        from paper_2409_08970_b200._native import check, lib

        torch = self.torch
        f32 = dtype == torch.float32
        pin_in = torch.from_numpy(np.ascontiguousarray(host.astype(np.float32 if f32 else np.float64))).pin_memory()
        n = cfg["n"]
        shape = (rows, sets, n) if cfg["op"] == "forward_all" else (rows, n)
        pin_out = torch.empty(shape, dtype=dtype).pin_memory()
        hin, hout = pin_in.numpy(), pin_out.numpy()
        sfx = "f32" if f32 else "f64"
        fn = {"forward": f"dctp_forward_host_{sfx}", "inverse": f"dctp_inverse_host_{sfx}",
              "forward_all": f"dctp_ensemble_forward_all_host_{sfx}", "chain": f"dctp_chain_forward_host_{sfx}"}
        f = getattr(lib, fn[cfg["op"]])

        def call():
            check(f(plan._h, C.c_void_p(hin.ctypes.data), C.c_void_p(hout.ctypes.data), rows))

        steps = max(3, min(self.args.steps, 10))
        for _ in range(2):
            call()
        self.barrier()
        t = time.perf_counter()
        for _ in range(steps):
            call()
        dt = self.max_over_ranks(time.perf_counter() - t)
        elem = 4 if f32 else 8
        batch = cfg["batch"]
        return {"value": batch * alg["out_samples"] * steps / dt, "unit": UNIT,
                "h2d_bytes_per_step": batch * n * elem, "d2h_bytes_per_step": batch * sets * n * elem,
                "path": f"{fn[cfg['op']]} (public C ABI, host buffers, pinned), synchronous per step, "
                        f"wall clock, max over ranks", "steps": steps}


def ctypes_ozaki_slices(n: int) -> int:
    import ctypes as C

    from paper_2409_08970_b200._native import check, lib

    s = C.c_int()
    check(lib.dctp_ozaki_slices(n, C.byref(s)))
    return s.value


def run_gpu_arm(args, rank, local, world):
    arm = GpuArm(args, rank, local, world)
    cfg = CONFIGS[args.config]
    head = arm.measure(args.config, headline=True)
    subs = {}
    if not args.no_configs:
        for key in ALL_BASELINE:
            subs[key] = head if key == args.config else arm.measure(key)
    do_cpu = rank == 0 and world == 1 and not args.no_cpu_baseline
    if do_cpu:
        head["cpu_baseline"] = cpu_baseline(cfg)
        for key, sub in subs.items():
            if sub is not head:
                sub["cpu_baseline"] = cpu_baseline(CONFIGS[key])
    if rank != 0:
        if world > 1:
            arm.torch.distributed.destroy_process_group()
        return
    sub_out = {}
    for key, sub in subs.items():
        sub_out[key] = {"workload": CONFIGS[key]["name"], "value": sub["value"], "unit": UNIT,
                        "ms_per_step": sub["ms_per_step"], "l2": sub["l2"], "roofline": sub["roofline"],
                        "e2e": sub["e2e"], "cpu_baseline": sub.get("cpu_baseline"), "kernels": sub["kernels"],
                        "setup_s": sub["setup_s"]}
    line = {
        "metric": METRIC, "value": head["value"], "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": max(3, args.warmup), "ms_per_step": head["ms_per_step"], "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": cfg["dtype"],
        "data": "synthetic: seeded reference Rng (mt19937_64 + Box-Muller) signals of the BASELINE config",
        "config": config_dict(cfg),
        "parallelism": f"batch sharded over {world} GPU(s), contiguous row slices, one plan per device, "
                       f"no data-path collective (gloo barriers / max only)",
        "l2": head["l2"], "setup_s": head["setup_s"],
        "roofline": head["roofline"], "clocks": head.get("clocks"), "sustained_load": head.get("sustained_load"),
        "e2e": head["e2e"], "gpu_launches": head["gpu_launches"], "kernels": head["kernels"],
        "cpu_baseline": head.get("cpu_baseline"),
        "configs": sub_out,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        arm.torch.distributed.destroy_process_group()


def main():
    args = parse()
    rank, local, world = dist_env()
    if args.config not in CONFIGS:
        raise SystemExit(f"unknown --config {args.config}; one of {sorted(CONFIGS)}")
    if args.impl == "reference":
        run_reference_arm(args, rank)
        return
    run_gpu_arm(args, rank, local, world)


if __name__ == "__main__":
    main()
