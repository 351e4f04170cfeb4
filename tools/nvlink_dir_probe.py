"""NVLink direction probe (diagnostic, not the bench contract).

Does the per-direction rate of a GPU pair drop when both directions carry
data at once, and does it matter whether the SMs pull (remote loads, a read
request travels against the data) or push (remote stores, posted)?  Times,
for GPUs 0 and 1 and `--gb` per direction:

  ce_uni / ce_bi       copy-engine peer copies (torch), one / both directions
  pull_uni / pull_bi   the fused pull kernel (rs_pull_spans) on the reader
                       GPU, sources in the peer's HBM
  push_uni / push_bi   the same kernel on the source GPU, destinations in the
                       peer's HBM (TMA tensor stores over NVLink)

    python tools/nvlink_dir_probe.py [--gb 4]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    from paper_2604_09107_b200 import ros
    ap = argparse.ArgumentParser()
    ap.add_argument("--gb", type=float, default=4.0)
    ap.add_argument("--items", type=int, default=16)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--digests", action="store_true", help="kernel writes its chunk-digest table")
    ap.add_argument("--only", default="", help="comma list of legs to run (default all)")
    a = ap.parse_args()
    n = int(a.gb * (1 << 30)) // a.items // 4096 * 4096
    total = n * a.items
    d = [torch.device("cuda", 0), torch.device("cuda", 1)]
    src = [torch.empty(total, dtype=torch.uint8, device=x) for x in d]
    dst = [torch.empty(total, dtype=torch.uint8, device=x) for x in d]
    for g in (0, 1):
        ros.synth_bf16(src[g], 11 + g)
        torch.cuda.synchronize(d[g])
    out = {"bytes_per_direction": total}

    def spans(t):
        base = t.data_ptr()
        return [base + i * n for i in range(a.items)]

    # copy engine
    def ce(dirs):
        streams = [torch.cuda.Stream(device=d[g]) for g in (0, 1)]
        for _ in range(2):
            for g in dirs:  # g: the receiving GPU
                with torch.cuda.stream(streams[g]):
                    dst[g].copy_(src[1 - g], non_blocking=True)
        for g in (0, 1):
            torch.cuda.synchronize(d[g])
        ev = {g: (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for g in dirs}
        for g in dirs:
            ev[g][0].record(streams[g])
        for _ in range(a.reps):
            for g in dirs:
                with torch.cuda.stream(streams[g]):
                    dst[g].copy_(src[1 - g], non_blocking=True)
        for g in dirs:
            ev[g][1].record(streams[g])
        for g in (0, 1):
            torch.cuda.synchronize(d[g])
        return [round(total * a.reps / (ev[g][0].elapsed_time(ev[g][1]) / 1e3) / 1e9, 1) for g in dirs]

    if not a.only or "ce" in a.only:
        out["ce_uni"] = ce([0])
        out["ce_bi"] = ce([0, 1])

    # fused kernel: pull (runs on the receiver) or push (runs on the sender).
    # Arguments are built once so the two directions' launches overlap (the
    # host does nothing between back-to-back calls but the ctypes call).
    import ctypes as C

    import numpy as np

    from paper_2604_09107_b200._lib import lib

    def kernel(dirs, push):
        res = {}
        reps = a.reps + 6
        args = {}
        nck = a.items * ((n // 4096 + 31) // 32 * 32)
        for g in dirs:
            s_ = np.asarray(spans(src[1 - g]), np.uint64)
            d_ = np.asarray(spans(dst[g]), np.uint64)
            l_ = np.asarray([n] * a.items, np.uint64)
            run_on = 1 - g if push else g
            od = torch.zeros(nck, dtype=torch.int64, device=d[run_on]) if a.digests else None
            args[g] = (s_, d_, l_, od)
        barrier = threading.Barrier(len(dirs))

        def one(g):  # g receives from 1-g
            run_on = 1 - g if push else g
            s_, d_, l_, od = args[g]
            odp = None if od is None else C.c_void_p(od.data_ptr())
            code, ms = C.c_int(), C.c_float()
            times = []
            barrier.wait()
            for _ in range(reps):
                rc = lib.rs_pull_spans(s_.ctypes.data, d_.ctypes.data, l_.ctypes.data, a.items, 4096,
                                       None, odp, run_on, None, C.byref(code), C.byref(ms))
                assert rc == 0 and code.value == 0, (rc, code.value)
                times.append(ms.value)
            mid = sorted(times[2:-2])  # the middle runs: both directions busy
            res[g] = round(total / (mid[len(mid) // 2] / 1e3) / 1e9, 1)

        ths = [threading.Thread(target=one, args=(g,)) for g in dirs]
        for t in ths:
            t.start()
        for t in ths:
            t.join()
        for g in dirs:
            assert torch.equal(dst[g].cpu()[:1 << 20], src[1 - g].cpu()[:1 << 20])
        return [res[g] for g in dirs]

    legs = {"pull_uni": ([0], False), "pull_bi": ([0, 1], False), "push_uni": ([0], True),
            "push_bi": ([0, 1], True)}
    for k, (dirs, push) in legs.items():
        if not a.only or k in a.only.split(","):
            out[k] = kernel(dirs, push)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
