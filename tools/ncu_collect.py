"""Collect the ncu --set full captures of tools/ncu_final.sh into one summary
(profiles/<round>/ncu_summary_final.json): per kernel the duration, DRAM traffic,
pipe activity and occupancy the rooflines in DESIGN.md quote.
usage: python tools/ncu_collect.py gpurun_out/ncu profiles/r02/ncu_summary.json"""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

METRICS = {
    "duration_us": ("gpu__time_duration.sum", {"ns": 1e-3, "us": 1, "usecond": 1, "ms": 1e3, "msecond": 1e3}),
    "dram_read_bytes": ("dram__bytes_read.sum", {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}),
    "dram_write_bytes": ("dram__bytes_write.sum", {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}),
    "sm_clock_ghz": ("gpc__cycles_elapsed.max.per_second", {"Ghz": 1, "Mhz": 1e-3}),
    "tensor_active_pct": ("sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", {"%": 1}),
    "tensor_active_pct_triage": ("TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", {"%": 1}),
    "dmma_active_pct": ("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", {"%": 1}),
    "fp64_pipe_pct": ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", {"%": 1}),
    "shared_pipe_pct": ("sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active", {"%": 1}),
    "tc_smem_wavefronts_pct": ("l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", {"%": 1}),
    "smem_bank_conflicts": ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", {"": 1}),
    "warps_active_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", {"%": 1}),
    "dram_throughput_pct": ("dram__throughput.avg.pct_of_peak_sustained_elapsed", {"%": 1}),
    "l2_to_l1_bytes": ("l1tex__m_xbar2l1tex_read_bytes.sum", {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9,
                                                              "Tbyte": 1e12}),
    "registers": ("launch__registers_per_thread", {"register/thread": 1, "": 1}),
    "grid": ("launch__grid_size", {"": 1}),
    "block": ("launch__block_size", {"": 1}),
}


def one(path: Path) -> dict:
    raw = subprocess.run(["ncu", "-i", str(path), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {h: (u, v) for h, u, v in zip(hdr, units, vals)}
    out = {"capture": path.name, "kernel": d.get("Kernel Name", ("", ""))[1][:160]}
    for key, (metric, scale) in METRICS.items():
        if metric in d:
            u, v = d[metric]
            try:
                out[key] = float(v.replace(",", "")) * scale.get(u, 1)
            except ValueError:
                pass
    out["dram_bytes"] = out.get("dram_read_bytes", 0) + out.get("dram_write_bytes", 0)
    return out


if __name__ == "__main__":
    src, dst = Path(sys.argv[1]), Path(sys.argv[2])
    res = [one(p) for p in sorted(src.glob("*.ncu-rep"))]
    dst.parent.mkdir(parents=True, exist_ok=True)
    dst.write_text(json.dumps(res, indent=1))
    for r in res:
        print(f"{r['capture']:28s} {r.get('duration_us', 0):9.1f} us  DRAM {r['dram_bytes'] / 1e6:8.1f} MB  "
              f"tensor {r.get('tensor_active_pct', r.get('tensor_active_pct_triage', 0)):5.1f}%  "
              f"dmma {r.get('dmma_active_pct', 0):5.1f}%  warps {r.get('warps_active_pct', 0):5.1f}%")
