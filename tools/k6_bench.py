"""K6 micro-benchmark: reference digest64 of one large span (diagnostic).
XXH64 is serial within a span, so this is the publish latency floor for the
largest item (Llama-3-8B embedding: 1.05 GB).

    python tools/k6_bench.py [--mb 1024]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    from paper_2604_09107_b200 import ros
    ap = argparse.ArgumentParser()
    ap.add_argument("--mb", type=int, default=1024)
    a = ap.parse_args()
    n = a.mb << 20
    t = torch.empty(n, dtype=torch.uint8, device="cuda:0")
    ros.synth_bf16(t, 5)
    torch.cuda.synchronize()
    ros.digest_spans([t.data_ptr()], [n], 0)
    best = None
    for _ in range(3):
        t0 = time.perf_counter()
        d = ros.digest_spans([t.data_ptr()], [n], 0)
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
    print(json.dumps({"bytes": n, "s": round(best, 4), "gbs": round(n / best / 1e9, 3),
                      "digest": hex(d[0])}))


if __name__ == "__main__":
    main()
