"""Both directions of a GPU pair through the ROS API in ONE process (peer
mappings, no IPC) -- the in-process twin of `bench.py --fanout ring` at
N=2 (diagnostic, not the bench contract).

Trainer t0 on GPU0 and t1 on GPU1; reader r1 on GPU1 pulls t0 while r0 on
GPU0 pulls t1, concurrently (two threads).  Prints per-direction GB/s
(median of the middle runs) for the workload's tensors.

    python tools/bidir_ros_probe.py [--workload llama3_8b] [--verify-off]
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

    import bench as B
    from paper_2604_09107_b200.ros import Cluster, Status
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="llama3_8b")
    ap.add_argument("--reps", type=int, default=8)
    ap.add_argument("--uni", action="store_true", help="one direction only")
    a = ap.parse_args()
    shapes = B.workload_shapes(a.workload)
    total = sum(2 * B._numel(s) for _, s in shapes)
    d = [torch.device("cuda", 0), torch.device("cuda", 1)]
    cl = Cluster()
    keep = []
    rd = {}
    for g in (0, 1):
        ta, tv = B.alloc_replica(shapes, d[g], seed_base=42 + 1000 * g)
        ra, rv = B.alloc_replica(shapes, d[1 - g])
        keep += [ta, ra]
        t = cl.open("m%d" % g, "trainer", 1)
        r = cl.open("m%d" % g, "reader", 1)
        for (n, v), (_, w) in zip(tv, rv):
            assert t.register_tensor(0, n, v) == Status.ok
            assert r.register_tensor(0, n, w) == Status.ok
        assert t.publish(1).status == Status.ok
        rd[g] = (r, ta, ra)
    res = {}
    dirs = [0] if a.uni else [0, 1]

    def run(g):
        r = rd[g][0]
        times = []
        for _ in range(a.reps):
            if r.is_published:
                r.unpublish()
            r.invalidate()
            assert r.replicate().status == Status.ok
            times.append(r.stats().last_pull_ms)
        mid = sorted(times[2:-2])
        res[g] = round(total / (mid[len(mid) // 2] / 1e3) / 1e9, 1)

    ths = [threading.Thread(target=run, args=(g,)) for g in dirs]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    for g in dirs:
        assert torch.equal(rd[g][1].cpu()[:1 << 24], rd[g][2].cpu()[:1 << 24])
    print(json.dumps({"workload": a.workload, "bytes": total, "dirs": dirs,
                      "per_direction_gbs": [res[g] for g in dirs]}))
    cl.close()


if __name__ == "__main__":
    main()
