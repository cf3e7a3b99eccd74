"""Condense one `ncu --set full` report into the JSON kept under profiles/.

  python tools/ncu_summary.py gpurun_out/x.ncu-rep '{"M":16400,"N":1536,"K":384}' > profiles/..json
"""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "gpu_time_us": ("gpu__time_duration.sum", "time"),
    "dram_bytes_read": ("dram__bytes_read.sum", None),
    "dram_bytes_write": ("dram__bytes_write.sum", None),
    "sm__pipe_tensor_cycles_active_pct": ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", 1),
    "xu_pipe_pct": ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", 1),
    "fma_pipe_pct": ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", 1),
    "issue_active_pct": ("smsp__issue_active.avg.pct_of_peak_sustained_active", 1),
    "lts_throughput_pct": ("lts__throughput.avg.pct_of_peak_sustained_elapsed", 1),
    "registers_per_thread": ("launch__registers_per_thread", 1),
    "threads_per_block": ("launch__block_size", 1),
    "grid": ("launch__grid_size", 1),
    "smem_per_block": ("launch__shared_mem_per_block_dynamic", 1),
}
UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1024, "MB": 1024 ** 2}


def main(rep, shape):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units, v = rows[0], rows[1], rows[2]
    d = dict(zip(h, v))
    u = dict(zip(h, units))
    out = {"kernel": d.get("Kernel Name", "").split("(")[0], "shape": json.loads(shape) if shape else None}
    for k, (m, scale) in KEYS.items():
        if m not in d:
            continue
        x = float(d[m].replace(",", ""))
        if scale is None:  # bytes: honour the unit column
            x *= UNITS.get(u.get(m, "byte"), 1)
            out[k] = int(x)
        elif scale == "time":
            x *= {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}.get(u.get(m, "usecond"), 1.0)
            out[k] = round(x, 3)
        else:
            out[k] = round(x * scale, 3) if scale != 1 else x
    stalls = {k.split("issue_stalled_")[1].split("_per_")[0]: float(d[k])
              for k in h if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")}
    out["top_stalls_per_issue"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:5])
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")
