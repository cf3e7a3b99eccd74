"""Wall time of the engine's pieces at the bench config: backbone graph alone, each head graph
alone, all heads together, and the full pipelined step (CUDA-event timed, graphs warmed)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2508_11584_b200.engine import VPEngine


def timed(fn, sync, reps=30):
    for _ in range(3):
        fn()
    sync()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    sync()
    return (time.perf_counter() - t) / reps * 1e3


def main():
    B = int(os.environ.get("VPE_BATCH", "16"))
    eng = VPEngine("vits14", 448, B)
    for _ in range(3):
        eng.submit()
    eng.synchronize()
    sp = eng.s_prod
    res = {}
    res["backbone"] = timed(lambda: eng._g_bb[0].launch(sp), eng.synchronize)
    for n in eng.heads:
        st = eng.s_head[n]
        res[n] = timed(lambda n=n, st=st: eng._g_head[(n, 0)].launch(st), eng.synchronize)

    def all_heads():
        for n in eng.heads:
            eng._g_head[(n, 0)].launch(eng.s_head[n])
    res["heads_concurrent"] = timed(all_heads, eng.synchronize)

    def serial():
        eng._g_bb[0].launch(sp)
        sp.sync()
        for n in eng.heads:
            eng._g_head[(n, 0)].launch(eng.s_head[n])
            eng.s_head[n].sync()
    res["serial_sum"] = timed(serial, eng.synchronize)
    res["pipelined_step"] = timed(eng.submit, eng.synchronize)
    print({k: round(v, 3) for k, v in res.items()})
    eng.close()


if __name__ == "__main__":
    main()
