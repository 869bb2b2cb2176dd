"""Summarise an ncu report (page raw) into the numbers the roofline needs.

usage: python tools/ncu_summary.py report.ncu-rep [algorithmic_bytes] [algorithmic_flops]
"""
import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "sm__cycles_elapsed.avg.per_second",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed.sum",
]


def summarise(path, alg_bytes=None, alg_flops=None):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        rec = {"kernel": d.get("Kernel Name", "")[:120]}
        for k in KEYS:
            if k in d:
                try:
                    rec[k] = float(d[k].replace(",", ""))
                except ValueError:
                    rec[k] = d[k]
                rec[k + ".unit"] = u.get(k, "")
        dur_ns = rec.get("gpu__time_duration.sum")
        tunit = {"ns": 1, "nsecond": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6}
        if dur_ns:
            dur_ns *= tunit.get(rec.get("gpu__time_duration.sum.unit"), 1)
        rb, wb = rec.get("dram__bytes_read.sum"), rec.get("dram__bytes_write.sum")
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
        if rb is not None:
            traffic = rb * scale.get(rec["dram__bytes_read.sum.unit"], 1) + \
                wb * scale.get(rec["dram__bytes_write.sum.unit"], 1)
            rec["dram_traffic_bytes"] = traffic
            if dur_ns:
                rec["dram_gbs"] = traffic / dur_ns
        if alg_bytes and dur_ns:
            rec["algorithmic_gbs"] = alg_bytes / dur_ns
        if alg_flops and dur_ns:
            rec["algorithmic_tflops"] = alg_flops / dur_ns / 1e3
        rec["duration_ns"] = dur_ns
        out.append(rec)
    return out


if __name__ == "__main__":
    ab = float(sys.argv[2]) if len(sys.argv) > 2 else None
    af = float(sys.argv[3]) if len(sys.argv) > 3 else None
    print(json.dumps(summarise(sys.argv[1], ab, af), indent=1))
