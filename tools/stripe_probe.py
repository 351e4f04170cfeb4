"""Fan-out shape probe: chain relays vs striped (scatter + all-gather) pulls
(diagnostic, not the bench contract).

N-1 receivers of one source's `--gb`, all flows at once, steady state (every
receiver already holds the bytes it forwards, so there is no chase):

  chain    receiver k pulls everything from k-1 (k=1 from the source)
  stripes  item i belongs to stripe i % (N-1); receiver k pulls its own
           stripe from the source and every other stripe from the receiver
           owning it (one fused kernel per receiver, spans from several GPUs)

Per receiver: GB/s of the fused pull kernel (rs_pull_spans, chunk verify off).
The NVLink accounting (a data byte costs ~1.125 on its direction plus ~0.19
of request traffic on the other) predicts ~686 for a chain relay and ~720 for
stripes at N=4.

    python tools/stripe_probe.py [--gb 4] [--gpus 4]
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import sys
import threading

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch

    from paper_2604_09107_b200 import ros
    from paper_2604_09107_b200._lib import lib
    ap = argparse.ArgumentParser()
    ap.add_argument("--gb", type=float, default=4.0)
    ap.add_argument("--gpus", type=int, default=4)
    ap.add_argument("--items", type=int, default=48)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    G = a.gpus
    R = G - 1
    n = int(a.gb * (1 << 30)) // a.items // 4096 * 4096
    total = n * a.items
    bufs = [torch.empty(total, dtype=torch.uint8, device=torch.device("cuda", g)) for g in range(G)]
    ros.synth_bf16(bufs[0], 5)
    for g in range(1, G):
        bufs[g].copy_(bufs[0].to(bufs[g].device))
    for g in range(G):
        torch.cuda.synchronize(g)
    lens = np.asarray([n] * a.items, np.uint64)

    def item(g, i):
        return bufs[g].data_ptr() + i * n

    def plan(shape):
        out = {}
        for k in range(1, G):
            if shape == "chain":
                srcs = [item(k - 1, i) for i in range(a.items)]
            else:
                srcs = [item(0, i) if i % R == k - 1 else item(i % R + 1, i) for i in range(a.items)]
            out[k] = (np.asarray(srcs, np.uint64), np.asarray([item(k, i) for i in range(a.items)], np.uint64))
        return out

    def run(shape):
        p = plan(shape)
        res = {}
        barrier = threading.Barrier(R)

        def one(k):
            s_, d_ = p[k]
            code, ms = C.c_int(), C.c_float()
            times = []
            barrier.wait()
            for _ in range(a.reps + 4):
                rc = lib.rs_pull_spans(s_.ctypes.data, d_.ctypes.data, lens.ctypes.data, a.items, 4096,
                                       None, None, k, None, C.byref(code), C.byref(ms))
                assert rc == 0 and code.value == 0, (rc, code.value)
                times.append(ms.value)
            mid = sorted(times[2:-2])
            res[k] = round(total / (mid[len(mid) // 2] / 1e3) / 1e9, 1)

        ths = [threading.Thread(target=one, args=(k,)) for k in range(1, G)]
        for t in ths:
            t.start()
        for t in ths:
            t.join()
        return [res[k] for k in range(1, G)]

    out = {"gpus": G, "bytes_per_receiver": total, "chain": run("chain"), "stripes": run("stripes")}
    for g in range(1, G):
        assert torch.equal(bufs[g][:1 << 22].cpu(), bufs[0][:1 << 22].cpu())
    print(json.dumps(out))


if __name__ == "__main__":
    main()
