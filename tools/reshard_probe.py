"""In-process multi-GPU TP=1 -> TP=2 reshard probe (diagnostic).

Trainer (TP=1) on cuda:0 publishes Llama-3-8B; a TP=2 reader replica has
shard 0 on cuda:1 and shard 1 on cuda:2 and replicates: both shards pull
their halves concurrently over NVLink (the trainer's egress is shared).
With --chain, a second TP=2 replica on cuda:3/cuda:1... chases the first.
Prints per-shard ingress GB/s and the replicate wall time.
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
    from paper_2604_09107_b200.ros import Cluster, Status, tp_slice
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="llama3_8b")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--reader-devs", default="1,2")
    a = ap.parse_args()
    shapes = B.workload_shapes(a.workload)
    devs = [int(x) for x in a.reader_devs.split(",")]
    t_arena, t_views = B.alloc_replica(shapes, torch.device("cuda:0"), seed_base=42)
    cl = Cluster()
    t = cl.open("m", "trainer", 1)
    r = cl.open("m", "tp2", 2)
    keep = []
    for (n, v), (_, shape) in zip(t_views, shapes):
        assert t.register_slice(0, n, v, tp_slice(shape, 2, None, 1, 0)) == Status.ok
        for s in range(2):
            geo = tp_slice(shape, 2, B.tp_dim(n), 2, s)
            buf = torch.empty(geo[3] * geo[5], dtype=torch.uint8, device=torch.device("cuda", devs[s]))
            keep.append((s, n, buf, geo, v))
            assert r.register_slice(s, n, buf, geo) == Status.ok
    assert t.publish(1).status == Status.ok
    shard_bytes = [sum(g[3] * g[5] for s2, _, _, g, _ in keep if s2 == s) for s in range(2)]
    walls, per_shard = [], []
    for k in range(a.steps + 1):
        if r.is_published:
            r.unpublish()
        r.invalidate()
        w0 = time.perf_counter()
        res = r.replicate()
        walls.append(time.perf_counter() - w0)
        assert res.status == Status.ok, res
    # verify against the trainer's slices
    for s, n, buf, (rows, w, r0, nr, c0, nc), v in keep:
        want = v.view(rows, w)[r0:r0 + nr, c0:c0 + nc].to(buf.device)
        assert torch.equal(buf.view(nr, nc), want), (s, n)
    st = r.stats()
    out = {"workload": a.workload, "shard_bytes": shard_bytes, "replicate_wall_s": walls[1:],
           "last_kernel_ms": st.last_pull_ms,
           "ingress_gbs_from_wall": [round(b / min(walls[1:]) / 1e9, 1) for b in shard_bytes],
           "verified": True}
    print(json.dumps(out))
    cl.close()


if __name__ == "__main__":
    main()
