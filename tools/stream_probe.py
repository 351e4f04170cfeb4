"""Off-box data plane probe (diagnostic): a reader pulls a published version
through the TCP stream server (loopback on one box), landing in pinned host
memory and through the pull kernel into device regions.

    python tools/stream_probe.py [--workload config1] [--reader-dev 1]
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

    import bench as B
    from paper_2604_09107_b200.ros import Cluster, Status
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="config1")
    ap.add_argument("--reader-dev", type=int, default=0)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    shapes = B.workload_shapes(a.workload)
    total = sum(2 * B._numel(s) for _, s in shapes)
    ta, tv = B.alloc_replica(shapes, torch.device("cuda:0"), seed_base=42)
    ra, rv = B.alloc_replica(shapes, torch.device("cuda", a.reader_dev))
    cl = Cluster()
    port = cl.listen()
    ep = f"tcp:127.0.0.1:{port}"
    t = cl.open("m", "trainer", 1)
    r = cl.open("m", "reader", 1)
    for (n, v), (_, x) in zip(tv, rv):
        t.register_tensor(0, n, v)
        r.register_tensor(0, n, x)
    t.set_endpoint(0, ep)
    assert t.publish(1).status == Status.ok
    walls, kms = [], []
    for _ in range(a.reps):
        if r.is_published:
            r.unpublish()
        r.invalidate()
        w0 = time.perf_counter()
        res = r.replicate()
        walls.append(time.perf_counter() - w0)
        assert res.status == Status.ok, res
        kms.append(r.stats().last_pull_ms)
    torch.cuda.synchronize()
    ok = torch.equal(ta.cpu(), ra.cpu())
    best = min(walls)
    print(json.dumps({"workload": a.workload, "bytes": total, "transport": "tcp loopback",
                      "wall_s_best": round(best, 4), "gbs_wall": round(total / best / 1e9, 2),
                      "kernel_ms": [round(k, 1) for k in kms], "bytes_equal": ok}))
    cl.close()


if __name__ == "__main__":
    main()
