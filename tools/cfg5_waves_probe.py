"""Config-5 wave probe: the 4096 problems in waves of P problems, each wave the
whole pipeline (norms -> plan -> draws -> split gather -> contraction), S
waves in flight on S streams of one CUDA graph.  A wave's M (P x 4 MB) is read
by the norm pass and again, from L2 if it is still there, by the gather.

  python tools/cfg5_waves_probe.py [P,S ...]     (default: a small sweep)
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import workloads  # noqa: E402
from paper_2105_04940_b200.pipeline import SketchPipeline, seeds_from_keys  # noqa: E402


def main():
    combos = [tuple(int(x) for x in a.split(",")) for a in sys.argv[1:]] or [
        (4096, 1), (256, 2), (64, 2), (32, 3), (16, 4), (16, 6), (8, 6), (8, 8)]
    torch.cuda.set_device(0)
    Md, Nd, sizes, B = bench.device_data(torch, "cfg5")
    m, n = Md.shape[-2:]
    p = Nd.shape[-1]
    K = len(sizes)
    W = 1024
    ref = SketchPipeline(m, n, p, sizes, W, "ONC", batch=B, dtype=torch.float32)
    keys = np.arange(B)
    CD_ref = ref.run(Md, Nd, seeds_from_keys("ONC", workloads.ROOT, (5, 1), keys, K)).clone()
    torch.cuda.synchronize()
    del ref
    for P, S in combos:
        nw = B // P
        pipes = [SketchPipeline(m, n, p, sizes, W, "ONC", batch=P, dtype=torch.float32) for _ in range(S)]
        out = torch.empty_like(CD_ref)
        # seeds: one buffer set per wave would be needed for the real thing; the probe
        # checks wave 0..S-1 only (each pipe's seeds = its first wave's)
        for s, q in enumerate(pipes):
            q.set_seeds(seeds_from_keys("ONC", workloads.ROOT, (5, 1), keys[s * P:(s + 1) * P], K))
        torch.cuda.synchronize()
        streams = [torch.cuda.Stream() for _ in range(S)]
        g = torch.cuda.CUDAGraph()

        def body():
            cap = torch.cuda.current_stream()
            for st in streams:
                st.wait_stream(cap)
            for w in range(nw):
                st, q = streams[w % S], pipes[w % S]
                with torch.cuda.stream(st):
                    r = q.launch(Md[w * P:(w + 1) * P], Nd[w * P:(w + 1) * P])
                    if w < S:
                        out[w * P:(w + 1) * P].copy_(r.view(P, m, p))
            for st in streams:
                cap.wait_stream(st)

        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            body()
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        with torch.cuda.graph(g):
            body()
        tcap = time.perf_counter() - t0
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ok = torch.equal(out[:S * P], CD_ref[:S * P])
        print(f"P={P:5d} S={S} waves={nw:5d}  step {np.median(ts):7.3f} ms (min {min(ts):.3f})  "
              f"capture {tcap:.1f} s  first waves bit-identical: {ok}", flush=True)
        del g, pipes, out
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
