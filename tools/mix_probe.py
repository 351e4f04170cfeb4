"""Mixed local + NVLink reshard pull, in one process on two GPUs (diagnostic).

The trainer is FSDP-2 (shard i = rows [i*R/2, (i+1)*R/2) of every tensor, on
cuda:i); a TP-2 reader pulls its shards resharded: shard s on cuda:s reads
most bytes from the local FSDP shard and the rest (the other half of the
row-parallel o/down projections) over NVLink from the peer.
--mode both: both reader shards pull at once (config 3 at N=2);
--mode one:  a reader holding only TP shard 0 pulls (the peer only serves).
Prints the pull-kernel time per reader shard and the bytes behind each link.
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

    import bench as B
    from paper_2604_09107_b200.ros import Cluster, Status, tp_slice
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="qwen25_32b")
    ap.add_argument("--mode", choices=["both", "one"], default="both")
    ap.add_argument("--steps", type=int, default=3)
    a = ap.parse_args()
    shapes = B.workload_shapes(a.workload)
    devs = [torch.device("cuda", i) for i in range(2)]
    cl = Cluster()
    t = cl.open("m", "trainer", 2)
    readers = [0, 1] if a.mode == "both" else [0]
    r = cl.open("m", "tp2", len(readers))
    keep = []
    for i, (n, shape) in enumerate(shapes):
        for s in range(2):
            g = tp_slice(shape, 2, 0, 2, s)
            w = torch.randint(0, 256, (g[3] * g[5],), dtype=torch.uint8, device=devs[s])
            keep.append(w)
            assert t.register_slice(s, n, w, g) == Status.ok
        for k, s in enumerate(readers):
            g = tp_slice(shape, 2, B.tp_dim(n), 2, s)
            buf = torch.empty(g[3] * g[5], dtype=torch.uint8, device=devs[s])
            keep.append(buf)
            assert r.register_slice(k, n, buf, g) == Status.ok, n
    streams = [torch.cuda.Stream(device=d) for d in devs]
    for k, s in enumerate(readers):
        r.set_stream(k, streams[s])
    assert t.publish(1).status == Status.ok
    out = []
    for step in range(a.steps + 1):
        if r.is_published:
            assert r.unpublish().status == Status.ok
        r.invalidate()
        res = r.replicate("latest")
        assert res.status == Status.ok, res
        st = r.stats()
        if step:
            out.append((st.fill_max_ms, st.fill_sum_ms, st.fill_bytes))
    ms = sum(o[0] for o in out) / len(out)
    print(json.dumps({"mode": a.mode, "fill_max_ms": round(ms, 3),
                      "fill_sum_ms": round(sum(o[1] for o in out) / len(out), 3),
                      "bytes_per_shard": out[0][2] // len(readers)}))


if __name__ == "__main__":
    main()
