"""Kernel microbenchmark of the fused pull (rs_pull_spans) against a plain
torch copy on the same bytes.  Diagnostic only (not the bench contract).

    python tools/kbench.py [--gb 4] [--chunks 4096,16384,65536]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    from paper_2604_09107_b200 import ros
    ap = argparse.ArgumentParser()
    ap.add_argument("--gb", type=float, default=4.0)
    ap.add_argument("--chunks", default="4096,16384,65536")
    ap.add_argument("--items", type=int, default=16)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    n = int(a.gb * (1 << 30)) // a.items // 256 * 256
    src = [torch.empty(n, dtype=torch.uint8, device=dev) for _ in range(a.items)]
    dst = [torch.empty(n, dtype=torch.uint8, device=dev) for _ in range(a.items)]
    for i, t in enumerate(src):
        ros.synth_bf16(t, 100 + i)
    total = n * a.items
    out = {"kernel": os.environ.get("RSB_PULL_KERNEL", "tma"), "bytes": total}
    # torch copy baseline
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(2):
        for s, d in zip(src, dst):
            d.copy_(s)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(a.reps):
        for s, d in zip(src, dst):
            d.copy_(s)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.reps
    out["torch_copy_ms"] = round(ms, 3)
    out["torch_copy_gbs_rw"] = round(2 * total / ms / 1e6, 1)
    sp = [t.data_ptr() for t in src]
    dp = [t.data_ptr() for t in dst]
    ls = [n] * a.items
    for chunk in [int(x) for x in a.chunks.split(",")]:
        nch = a.items * ((n + chunk - 1) // chunk)
        dig = torch.empty(nch, dtype=torch.int64, device=dev)
        for mode in ("copy", "hash"):
            best = 1e9
            for r in range(a.reps + 2):
                code, kms = ros.pull_spans(sp, dp if mode == "copy" else None, ls, chunk, None, dig, 0)
                assert code == 0
                if r >= 2:
                    best = min(best, kms)
            moved = (2 if mode == "copy" else 1) * total
            out[f"{mode}_c{chunk}_ms"] = round(best, 3)
            out[f"{mode}_c{chunk}_gbs"] = round(moved / best / 1e6, 1)
        # verify mode: expect table = computed digests
        best = 1e9
        for r in range(a.reps + 2):
            code, kms = ros.pull_spans(sp, dp, ls, chunk, dig, None, 0)
            assert code == 0
            if r >= 2:
                best = min(best, kms)
        out[f"verify_c{chunk}_ms"] = round(best, 3)
        out[f"verify_c{chunk}_gbs"] = round(2 * total / best / 1e6, 1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
