"""Diagnostics: run the engine step N times on the same frame and report which outputs differ
bitwise from the first run (ring taps, depth, seg labels, det boxes/scores), with programmatic
dependent launch on (VPEngine(pdl=True)) or off; then the latency-mode p50 per head.

  VPE_BATCH=1 REPS=200 PDL=1 python tools/pdl_determinism.py"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2508_11584_b200.engine import VPEngine
from paper_2508_11584_b200.weights import make_frames

B = int(os.environ.get("VPE_BATCH", "1"))
pdl = os.environ.get("PDL", "1") == "1"
eng = VPEngine("vits14", 448, B, pdl=pdl)
eng.pixels.copy_(make_frames(B, 448, 0).to(eng.device))
eng.channel.register_consumer(99)


def grab():
    eng.submit()
    eng.synchronize()
    out = {}
    for head, d in eng.out.items():
        for k, v in d.items():
            if torch.is_tensor(v):
                out[f"{head}.{k}"] = v.clone()
    lease = eng.channel.acquire_latest(99)
    if lease is not None:
        for lab, v in eng.channel.view(lease).items():
            out[f"tap.{lab}"] = v.clone()
        eng.channel.commit(lease)
    return out


ref = grab()
bad = 0
reps = int(os.environ.get("REPS", "200"))
for i in range(reps):
    o = grab()
    diff = [k for k, v in o.items() if k in ref and not torch.equal(v, ref[k])]
    if diff:
        bad += 1
        print(f"run {i}: differs in {diff}")
print(f"pdl={pdl} batch={B}: {bad} of {reps} replays differ bitwise ({len(ref)} tensors compared)")
for _ in range(5):
    eng.submit()
eng.synchronize()
eng.latencies_ms()
for _ in range(100):
    eng.submit(record_latency=True)
    eng.synchronize()
lat = eng.latencies_ms()
print("p50 ms:", {n: round(statistics.median(v), 4) for n, v in lat.items() if v})
eng.close()
