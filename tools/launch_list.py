"""One pipelined C2 engine step (batch 16) bracketed by cudaProfilerStart/Stop, for
`ncu --profile-from-start off --metrics gpu__time_duration.sum ... python tools/launch_list.py`;
then `python tools/launch_list.py --summarize gpurun_out/x.csv` aggregates per kernel."""
import collections
import csv
import os
import re
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def summarize(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    rows = [h] + [r for r in rows[1:] if r[h.index("Metric Name")] == "gpu__time_duration.sum"]
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}[rows[1][ui]]
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        nm = re.sub(r"\(.*", "", r[ki])[:64]
        agg[nm][0] += 1
        agg[nm][1] += float(r[vi].replace(",", "")) * scale
    tot = sum(v[1] for v in agg.values())
    print(f"{len(rows) - 1} launches, {tot:.1f} us serialised")
    for nm, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{t:9.1f} us {c:4d} {t / c:8.2f} us/launch {100 * t / tot:5.1f}%  {nm}")


def main():
    import torch
    from paper_2508_11584_b200.engine import VPEngine
    B = int(os.environ.get("VPE_BATCH", "16"))
    eng = VPEngine("vits14", 448, B)
    for _ in range(4):
        eng.submit()
    eng.synchronize()
    torch.cuda.cudart().cudaProfilerStart()
    eng.submit()
    eng.synchronize()
    torch.cuda.cudart().cudaProfilerStop()
    eng.close()


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[1] == "--summarize":
        summarize(sys.argv[2])
    else:
        main()
