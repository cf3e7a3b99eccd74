"""ncu target: every kernel class bench.py times (kernel_rooflines) launched ONCE each at the bench
config, bracketed by cudaProfilerStart/Stop; then `--summarize` turns the raw CSV into
profiles/round2_ncu_<class>.json (shape, duration, DRAM bytes, pipe utilisation), which bench.py
reads for `roofline.traffic`.

  ncu --set full --clock-control none --profile-from-start off -o gpurun_out/cls \\
      python tools/ncu_classes.py > gpurun_out/cls_order.json
  ncu -i gpurun_out/cls.ncu-rep --page raw --csv > gpurun_out/cls_raw.csv
  python tools/ncu_classes.py --summarize gpurun_out/cls_raw.csv gpurun_out/cls_order.json"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

METRICS = {"duration_us": ("gpu__time_duration.sum", 1e-3), "dram_bytes_read": ("dram__bytes_read.sum", 1.0),
           "dram_bytes_write": ("dram__bytes_write.sum", 1.0),
           "tensor_pct": ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", 1.0),
           "dram_pct": ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
           "issue_pct": ("smsp__issue_active.avg.pct_of_peak_sustained_active", 1.0)}


def summarize(raw_csv, order_json):
    rows = list(csv.reader(open(raw_csv)))
    h, units = rows[0], rows[1]
    order = json.loads([l for l in open(order_json).read().splitlines() if l.startswith('[')][-1])
    kern = [r for r in rows[2:] if len(r) == len(h) and " at::" not in r[h.index("Kernel Name")]]  # drop torch fills
    # match each class to the next profiled kernel of its name (other kernels in the range, e.g.
    # the seg head run that produces the seg class's input logits, are skipped)
    pairs, k = [], 0
    for cls in order:
        base = cls["kernel"].split("<")[0].split(" ")[0]
        while k < len(kern) and base not in kern[k][h.index("Kernel Name")]:
            k += 1
        if k == len(kern):
            print(f"warning: no profiled kernel for {cls['class']}")
            break
        pairs.append((kern[k], cls))
        k += 1
    for r, cls in pairs:
        d = {"class": cls["class"], "kernel": r[h.index("Kernel Name")], "shape": cls["shape"],
             "source": "ncu --set full --clock-control none, one cold launch (tools/ncu_classes.py)"}
        for k, (m, sc) in METRICS.items():
            if m in h:
                v = float(r[h.index(m)].replace(",", ""))
                u = units[h.index(m)]
                if m.startswith("dram__bytes"):
                    sc = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[u]
                if m == "gpu__time_duration.sum":
                    sc = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}[u]
                d[k] = v * sc
        d["dram_bytes_read"] = int(d.get("dram_bytes_read", 0))
        d["dram_bytes_write"] = int(d.get("dram_bytes_write", 0))
        with open(os.path.join(ROOT, "profiles", f"round2_ncu_{cls['class']}.json"), "w") as f:
            json.dump(d, f, indent=1)
        print(cls["class"], d["kernel"][:50], f"{d.get('duration_us', 0):.1f} us",
              f"dram {(d['dram_bytes_read'] + d['dram_bytes_write']) / 1e6:.1f} MB")


def main():
    import torch

    import bench
    from paper_2508_11584_b200.engine import VPEngine

    eng = VPEngine("vits14", 448, 16)
    for _ in range(eng.capacity + 1):  # every ring slot holds a real frame (the seg class reads one)
        eng.submit()
    eng.synchronize()
    order = []

    def once(fn, reps=0, replays=0):
        fn()
        torch.cuda.synchronize()
        return 1.0

    bench._graph_time = once
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStart()
    _, out = bench.kernel_rooflines(eng, {"tensor": 1.0, "hbm": 1.0})
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()
    order = [{"class": r["class"], "shape": r["shape"], "kernel": r["kernel"]} for r in out]
    print(json.dumps(order))


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--summarize":
        summarize(sys.argv[2], sys.argv[3])
    else:
        main()
