#!/usr/bin/env python3
"""Benchmark of the B200 Fast DCT+ apply path (the driver's contract).

Workload (BASELINE.json configs[1], the config its metric is quoted on):
  C2 — path graph n = 256, edge (127,128) reweighted 1.0 -> 0.3, i.e.
  RankOneUpdate::edge_delta(128, 129, -0.7) (1-based); forward DCT+ of a batch
  of 65536 fp64 signals, AR(1) rows (rho = 0.95, unit innovation) drawn with
  the reference's Rng (signal.hpp:18-55) from mix_seed(2409, 256, 2).
A step = one forward DCT+ of the whole batch.  Metric: transformed (output)
samples per second, whole job.  The other BASELINE configs are parity cases
(tests/test_gpu_parity.py); `--config K` benches another one for development.

Arms:
  default            this repo's sm_100a kernels through the C ABI.
  --impl reference   the reference's own CPU implementation (oracle/_ref,
                     the unmodified headers compiled here) on all host
                     cores, same metric / config, bounded sample per step.

Multi-GPU (torchrun): every rank transforms its own 65536-signal batch (weak
scaling, no data-path collective — signals are independent); the timing is
the max over ranks of a barrier-bracketed CUDA-event interval.
"""
from __future__ import annotations

import argparse
import json
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
FP64_PEAK_FILE = ROOT / "profiles" / "peaks_fp64.json"
L2_BYTES = 126 * 2**20


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", type=int, default=2, help="BASELINE config id (2 = the headline workload; 6 = rank-k chain, 7-8 = NFST route, SURVEY 8f)")
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))


# ------------------------------------------------------------------ workloads

def workload(cid: int):
    from paper_2409_08970_b200.configs import WORKLOADS

    return WORKLOADS[cid]


def describe(cfg) -> dict:
    return {"workload": cfg.name, "n": cfg.n, "batch_per_gpu": cfg.batch,
            "precision": cfg.dtypes[0], "output_sets": 16 if cfg.progressive else 1}


def api_name(cfg) -> str:
    if cfg.chain:
        return "chain_forward"
    return "PrunedEnsemblePlan::forward_all" if cfg.progressive else "DctPlusPlan::forward"


def algorithmic(cfg, plan) -> dict:
    """bytes = elem * n * (1 + K_out); flops = 2.5 n log2 n +
    2 * n_kept * n_active * K (the direct Cauchy stage, per signal)."""
    elem = 4 if cfg.dtypes[0] == "f32" else 8
    kout = 16 if cfg.progressive else 1
    if cfg.chain:  # one dense product with the composed basis, no DCT
        return {"bytes": elem * cfg.n * 2, "flops_cauchy": 2.0 * cfg.n * cfg.n, "flops_dct": 0.0,
                "out_samples": cfg.n}
    if cfg.progressive:
        cauchy = sum(2 * m.n_kept * m.n_active for m in (plan.member(r) for r in range(1, 17)))
    else:
        cauchy = 2 * plan.n_kept * plan.n_active
    dct = 2.5 * cfg.n * np.log2(cfg.n)
    return {"bytes": elem * cfg.n * (1 + kout), "flops_cauchy": float(cauchy), "flops_dct": float(dct),
            "out_samples": cfg.n * kout}


# ---------------------------------------------------------------------- clocks

class ClockSampler:
    """nvidia-smi-equivalent sampling through NVML during the timed region."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, index: int):
        self.samples, self.reasons = [], set()
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
                mask = self.nvml.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if mask & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.002)

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
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ----------------------------------------------------------------- CPU arms

def cpu_reference_rate(cfg, signals: np.ndarray, threads: int = 0, passes: int = 2):
    """The reference's own CPU DctPlusPlan::forward / forward_all (oracle/_ref)
    over `signals`, all host threads; min of `passes` (bench.hpp:156-162)."""
    from oracle import checkers as O
    from paper_2409_08970_b200.configs import general_direction

    ref = O.Reference()
    ups = [O.Update(k, rho, i, j, tuple(general_direction(cfg.n)) if k == 2 else None)
           for (k, rho, i, j) in cfg.updates]
    if cfg.chain:
        obj = ref.chain(cfg.n, ups)
        run = lambda: obj.forward(signals, threads=threads)  # noqa: E731
    elif cfg.progressive:
        obj = ref.ensemble(cfg.n, ups, cfg.n, float(np.finfo(np.float64).max))
        run = lambda: obj.forward_all(signals, threads=threads)  # noqa: E731
    else:
        obj = ref.plan(cfg.n, ups[0])
        run = lambda: obj.forward(signals, threads=threads)  # noqa: E731
    best = float("inf")
    for _ in range(passes):
        t = time.perf_counter()
        run()
        best = min(best, time.perf_counter() - t)
    return best


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


def sample_size(cfg, threads: int, target_s: float) -> tuple:
    """Signals for ~target_s of reference CPU work (probe on a small slice)."""
    import paper_2409_08970_b200 as P

    probe = min(cfg.batch, max(64, 16 * threads))
    sig = P.fill_signals(cfg.seed, cfg.dist, cfg.n, probe, cfg.r)
    dt = cpu_reference_rate(cfg, sig, threads, passes=1)
    per = dt / probe
    rows = int(min(cfg.batch, max(probe, target_s / max(per, 1e-9))))
    return rows, per


def run_reference_arm(args, cfg, rank: int):
    if rank != 0:
        return
    import paper_2409_08970_b200 as P

    threads = host_cores()
    rows, _ = sample_size(cfg, threads, target_s=max(1.0, 120.0 / max(1, args.steps + args.warmup)))
    sig = P.fill_signals(cfg.seed, cfg.dist, cfg.n, rows, cfg.r)
    alg_out = cfg.n * (16 if cfg.progressive else 1)
    for _ in range(args.warmup):
        cpu_reference_rate(cfg, sig, threads, passes=1)
    times = [cpu_reference_rate(cfg, sig, threads, passes=1) for _ in range(args.steps)]
    total = sum(times)
    value = rows * alg_out * args.steps / total
    line = {
        "impl": "reference", "metric": "DCT+ transformed samples/sec", "value": value,
        "unit": "samples/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (reference Rng, seeded)",
        "config": {**describe(cfg), "sample_signals_per_step": rows},
        "cpu_baseline": {"value": value, "unit": "samples/s", "cores": threads, "kind": "reference",
                         "sample": f"{rows} of {cfg.batch} signals per step, reference {api_name(cfg)} "
                                   f"(oracle/_ref, FFTW stand-in), {threads} threads on {cpu_model()}"},
        "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------- GPU arm

def fp64_peak():
    try:
        return json.loads(FP64_PEAK_FILE.read_text())
    except Exception:
        return None


def run_gpu_arm(args, cfg, rank: int, local: int, world: int):
    import torch

    import paper_2409_08970_b200 as P
    from paper_2409_08970_b200.configs import make_plan

    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)

    t0 = time.perf_counter()
    plan = make_plan(cfg, device=local)
    setup_s = time.perf_counter() - t0

    dtype = torch.float32 if cfg.dtypes[0] == "f32" else torch.float64
    host = P.fill_signals(P.mix_seed(2409, cfg.n, cfg.cid) + rank, cfg.dist, cfg.n, cfg.batch, cfg.r)
    x = torch.as_tensor(host, device=dev).to(dtype)
    sets = 17 if cfg.progressive else 1
    y = torch.empty((cfg.batch, sets, cfg.n) if cfg.progressive else (cfg.batch, cfg.n), dtype=dtype, device=dev)

    def step():
        if cfg.progressive:
            plan.forward_all_batch(x, sync=False, out=y)
        else:
            plan.forward(x, sync=False, out=y)

    alg = algorithmic(cfg, plan)
    stream = torch.cuda.current_stream(dev)

    def barrier():
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize(dev)

    for _ in range(max(3, args.warmup)):
        step()
    plan.sync_check() if not cfg.progressive else None
    barrier()

    # timed region: K steps, CUDA events on the launching stream, per-kernel events on
    P.profile_reset()
    P.profile_enable(True)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        barrier()
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        barrier()
        # keep the sampler alive across a second identical interval so short
        # runs still see load-state clocks
        for _ in range(args.steps):
            step()
        torch.cuda.synchronize(dev)
    P.profile_enable(False)
    prof = P.profile_summary()
    ms = ev0.elapsed_time(ev1)
    if world > 1:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    ms_per_step = ms / args.steps
    total_samples = cfg.batch * alg["out_samples"] * world * args.steps
    value = total_samples / (ms * 1e-3)

    # per-kernel roofline (the dominant kernel of the step); the profile
    # covered 2*K steps, so per-launch averages are over 2*K launches
    launches = {k: v[0] for k, v in prof.items()}
    per_launch_ms = {k: v[1] / max(v[0], 1) for k, v in prof.items()}
    top = max(per_launch_ms, key=per_launch_ms.get)
    gpu_launches = sum(launches.values()) // 2
    peaks = json.loads(MEASURED.read_text()) if MEASURED.exists() else {}
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    hbm_src = "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else "B200_PROFILING.md fallback 6650 GB/s"
    fp = fp64_peak() or {}
    f32 = cfg.dtypes[0] == "f32"
    # The dominant kernel's algorithmic work per launch: the
    # direct Cauchy stage 2 * n_kept * n_active (* K members) plus 2.5 n log2 n
    # for the DCT, per signal; bytes = elem * n * (1 + K_out) per signal.
    # A product kernel (Cauchy stage, folded W product, dense basis, chain,
    # progressive SGEMM) is rated on the Cauchy-stage flops over its own
    # launch time; the fused kernel also carries the DCT; any other top
    # kernel falls back to the whole step.
    product = any(k in top for k in ("cauchy", "fold_w", "dense", "chain", "progressive_sgemm", "progressive_tc32"))
    if "fused" in top:
        flops, t_ms = (alg["flops_cauchy"] + alg["flops_dct"]) * cfg.batch, per_launch_ms[top]
    elif product:
        flops, t_ms = alg["flops_cauchy"] * cfg.batch, per_launch_ms[top]
    else:
        flops, t_ms = (alg["flops_cauchy"] + alg["flops_dct"]) * cfg.batch, ms_per_step
    nbytes = alg["bytes"] * cfg.batch
    if f32 and "tc32" in top:
        # tcgen05 kind::tf32 with the 3xTF32 split: three tensor-core products
        # per algorithmic one; dense TF32 runs at half the bf16 rate
        tf = fp.get("tcgen05_tf32_tflops")
        bf = peaks.get("bf16_tflops")
        if tf:
            peak = tf / 3.0
            src = "profiles/peaks_fp64.json tcgen05_tf32_tflops (tools/tc_peak.cu, measured) / 3 (3xTF32 passes)"
        else:
            peak = bf / 2.0 / 3.0 if bf else None
            src = "MEASURED_PEAKS.json bf16_tflops / 2 (dense TF32 rate) / 3 (3xTF32 passes)"
        bound = "tensor"
    elif f32:
        peak = max(fp.get("fp32_fma_tflops") or 0.0, fp.get("fp32_ffma2_tflops") or 0.0) or None
        src = "profiles/peaks_fp64.json max(fp32_fma_tflops, fp32_ffma2_tflops) (tools/peaks.cu, measured)"
        bound = "fp32-fma"
    else:
        peak = max(fp.get("dmma_m8n8k4_tflops") or 0.0, fp.get("dmma_m16n8k16_tflops") or 0.0) or None
        src = "profiles/peaks_fp64.json max DMMA m8n8k4 / m16n8k16 (tools/peaks.cu, measured fp64 tensor-core peak)"
        bound = "tensor"
    achieved = flops / (t_ms * 1e-3) / 1e12
    hbm_achieved = nbytes / (t_ms * 1e-3) / 1e9
    t_flop = flops / (peak * 1e12) if peak else 0.0
    t_hbm = nbytes / (hbm_peak * 1e9)
    if "nfst" in top:
        # the NFST route's work is O(n log n) per signal (four FFTs of <= n
        # points and a 35-tap gather per root): its roofline is the HBM
        # traffic of one read and one write per sample
        t_ms = per_launch_ms[top]
        hbm_achieved = nbytes / (t_ms * 1e-3) / 1e9
        achieved, t_flop = 0.0, 0.0
    if t_hbm >= t_flop:
        roof = {"bound": "hbm", "kernel": top, "achieved": hbm_achieved, "peak": hbm_peak, "unit": "GB/s",
                "frac": hbm_achieved / hbm_peak, "traffic": None, "peak_source": hbm_src}
    else:
        roof = {"bound": bound, "kernel": top, "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                "frac": (achieved / peak) if peak else None, "traffic": None, "peak_source": src}
    roof.update({"algorithmic_flops_per_launch": flops, "algorithmic_bytes_per_launch": nbytes,
                 "launch_ms": t_ms, "kernel_share_of_step": t_ms / ms_per_step,
                 "hbm_achieved_gbs": hbm_achieved, "hbm_frac": hbm_achieved / hbm_peak,
                 "compute_achieved_tflops": achieved, "compute_frac": (achieved / peak) if peak else None,
                 "t_roof_ms": max(t_flop, t_hbm) * 1e3})
    # DRAM traffic of the dominant kernel from the committed ncu --set full capture
    # of this workload (profiles/traffic.json), per launch like `achieved`
    tfile = ROOT / "profiles" / "traffic.json"
    tmap = json.loads(tfile.read_text()) if tfile.exists() else {}
    rec = tmap.get(cfg.name)
    if rec and rec.get("kernel") == top:
        roof["traffic"] = rec["dram_bytes_per_launch"]
        roof["traffic_source"] = rec["source"]
    roof["step_hbm_gbs"] = alg["bytes"] * cfg.batch / (ms_per_step * 1e-3) / 1e9
    roof["step_hbm_frac"] = roof["step_hbm_gbs"] / hbm_peak

    # end to end through the public API with host buffers (pinned), per step:
    # H2D of the inputs, the transform, D2H of the coefficients
    e2e_steps = args.e2e_steps or max(3, min(args.steps, 10))
    pinned_in = torch.from_numpy(host.astype(np.float32 if dtype == torch.float32 else np.float64)).pin_memory()
    out_shape = (cfg.batch, sets, cfg.n) if cfg.progressive else (cfg.batch, cfg.n)
    pinned_out = torch.empty(out_shape, dtype=dtype).pin_memory()
    hin, hout = pinned_in.numpy(), pinned_out.numpy()

    # the public host-buffer entry (what DctPlusPlan.forward(numpy) calls), on pinned buffers
    import ctypes as C

    from paper_2409_08970_b200._native import check, lib

    def e2e_call():
        if cfg.chain:
            fn = lib.dctp_chain_forward_host_f32 if dtype == torch.float32 else lib.dctp_chain_forward_host_f64
        elif cfg.progressive:
            fn = lib.dctp_ensemble_forward_all_host_f32 if dtype == torch.float32 else lib.dctp_ensemble_forward_all_host_f64
        else:
            fn = lib.dctp_forward_host_f32 if dtype == torch.float32 else lib.dctp_forward_host_f64
        check(fn(plan._h, C.c_void_p(hin.ctypes.data), C.c_void_p(hout.ctypes.data), cfg.batch))

    for _ in range(2):
        e2e_call()
    barrier()
    t = time.perf_counter()
    for _ in range(e2e_steps):
        e2e_call()
    e2e_s = time.perf_counter() - t
    if world > 1:
        tt = torch.tensor([e2e_s], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        e2e_s = float(tt.item())
    e2e_value = cfg.batch * alg["out_samples"] * world * e2e_steps / e2e_s
    elem = 4 if dtype == torch.float32 else 8

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            threads = host_cores()
            rows, _ = sample_size(cfg, threads, target_s=4.0)
            sig = P.fill_signals(cfg.seed, cfg.dist, cfg.n, rows, cfg.r)
            dt = cpu_reference_rate(cfg, sig, threads, passes=2)
            cpu = {"value": rows * alg["out_samples"] / dt, "unit": "samples/s", "cores": threads, "kind": "reference",
                   "sample": f"{rows} of {cfg.batch} signals, reference "
                             f"{api_name(cfg)} (oracle/_ref, FFTW stand-in), "
                             f"min of 2 passes, {threads} threads on {cpu_model()}"}
        except Exception as e:  # reference not built on this box
            cpu = {"value": None, "unit": "samples/s", "cores": 0, "kind": "reference", "sample": f"unavailable: {e}"}

    if rank == 0:
        line = {
            "metric": "DCT+ transformed samples/sec", "value": value, "unit": "samples/s", "n_gpus": world,
            "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": cfg.dtypes[0],
            "data": "synthetic: seeded reference Rng (mt19937_64 + Box-Muller) signals of the BASELINE config",
            "config": {**describe(cfg), "parallelism": f"batch-sharded x{world} (no collective)",
                       "l2": f"inputs {cfg.batch * cfg.n * elem / 2**20:.0f} MiB per step > 126 MB L2 with the "
                             f"{cfg.batch * alg['out_samples'] * elem / 2**20:.0f} MiB output: no flush needed"
                       if cfg.batch * cfg.n * elem * 2 > L2_BYTES else "inputs fit in L2 (small config)",
                       "setup_s": setup_s},
            "roofline": roof,
            "clocks": clocks.report(),
            "e2e": {"value": e2e_value, "unit": "samples/s", "h2d_bytes_per_step": cfg.batch * cfg.n * elem,
                    "d2h_bytes_per_step": cfg.batch * alg["out_samples"] * elem,
                    "path": "public API with host buffers (pinned), synchronous per step", "steps": e2e_steps},
            "gpu_launches": gpu_launches,
            "kernels": {k: {"launches_per_step": launches[k] / (2 * args.steps), "ms_per_launch": per_launch_ms[k]}
                        for k in launches},
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def main():
    args = parse()
    rank, local, world = dist_env()
    cfg = workload(args.config)
    if args.impl == "reference":
        run_reference_arm(args, cfg, rank)
        return
    run_gpu_arm(args, cfg, rank, local, world)


if __name__ == "__main__":
    main()
