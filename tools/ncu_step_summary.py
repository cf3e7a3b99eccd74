"""Condense the raw ncu --set full page of one engine step (tools/ncu_step.sh) into the per-kernel
and per-class JSON kept under profiles/ (NS-1 evidence: tensor-pipe utilisation for the
contractions, achieved DRAM GB/s for the memory-bound kernels; times are ncu's serialised,
cold-cache replays: read shares and counters, not absolute step time).

  python tools/ncu_step_summary.py gpurun_out/step_full_r2b_raw.csv.gz > profiles/round2_ncu_step.json
"""
import collections
import csv
import gzip
import io
import json
import re
import sys

M = {
    "time_us": "gpu__time_duration.sum",
    "dram_read": "dram__bytes_read.sum",
    "dram_write": "dram__bytes_write.sum",
    "tensor_pct": "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "xu_pct": "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "fma_pct": "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "issue_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "l2_pct": "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm_busy_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "regs": "launch__registers_per_thread",
    "block": "launch__block_size",
    "grid": "launch__grid_size",
    "smem_dyn": "launch__shared_mem_per_block_dynamic",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1024, "MB": 1024 ** 2, "GB": 1024 ** 3,
         "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "ns": 1e-3, "us": 1.0, "ms": 1e3}


def load(path):
    op = gzip.open if path.endswith(".gz") else open
    with op(path, "rt") as f:
        rows = list(csv.reader(io.StringIO(f.read())))
    h, units = rows[0], rows[1]
    return h, units, rows[2:]


def main(path):
    h, units, rows = load(path)
    idx = {k: h.index(v) for k, v in M.items() if v in h}
    kernels = []
    for r in rows:
        if len(r) != len(h):
            continue
        name = re.sub(r"\(.*", "", r[h.index("Kernel Name")]).replace("void ", "").strip()
        d = {"kernel": name}
        for k, i in idx.items():
            v = r[i].replace(",", "")
            try:
                x = float(v)
            except ValueError:
                continue
            u = units[i]
            if k in ("time_us", "dram_read", "dram_write"):
                x *= SCALE.get(u, 1)
            d[k] = x
        kernels.append(d)
    tot = sum(k.get("time_us", 0) for k in kernels)
    cls = collections.OrderedDict()
    for k in kernels:
        c = cls.setdefault(k["kernel"], {"launches": 0, "time_us": 0.0, "dram_bytes": 0.0, "_w": collections.Counter()})
        c["launches"] += 1
        t = k.get("time_us", 0)
        c["time_us"] += t
        c["dram_bytes"] += k.get("dram_read", 0) + k.get("dram_write", 0)
        for m in ("tensor_pct", "xu_pct", "fma_pct", "issue_pct", "dram_pct", "l2_pct"):
            if m in k:
                c["_w"][m] += k[m] * t
    out = []
    for name, c in sorted(cls.items(), key=lambda kv: -kv[1]["time_us"]):
        t = c["time_us"]
        row = {"kernel": name, "launches": c["launches"], "time_us": round(t, 2), "share": round(t / tot, 4),
               "us_per_launch": round(t / c["launches"], 2),
               "dram_bytes_per_launch": int(c["dram_bytes"] / c["launches"]),
               "dram_gbs": round(c["dram_bytes"] / (t * 1e-6) / 1e9, 1) if t else None}
        for m in ("tensor_pct", "xu_pct", "fma_pct", "issue_pct", "dram_pct", "l2_pct"):
            if c["_w"][m]:
                row[m] = round(c["_w"][m] / t, 1)
        out.append(row)
    print(json.dumps({"source": path, "launches": len(kernels), "serialised_us": round(tot, 1),
                      "note": "ncu --set full --clock-control none, one pipelined C2 step (batch 16); "
                              "time-weighted averages per kernel class; serialised cold-cache replays",
                      "classes": out, "kernels": kernels}, indent=1))


if __name__ == "__main__":
    main(sys.argv[1])
