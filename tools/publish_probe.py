"""Publish latency probe (diagnostic): the trainer republishes Llama-3-8B a
few times; prints each publish's device time (K6 item digests, group
packing, chunk-digest pass) and wall time."""
from __future__ import annotations

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
    dev = torch.device("cuda", 0)
    shapes = B.workload_shapes("llama3_8b")
    arena, views = B.alloc_replica(shapes, dev, seed_base=42)
    torch.cuda.synchronize()
    cl = Cluster()
    t = cl.open("m", "trainer", 1)
    for n, v in views:
        assert t.register_tensor(0, n, v) == Status.ok
    out = []
    for v in range(1, 6):
        if v > 1:
            assert t.unpublish().status == Status.ok
        w0 = time.perf_counter()
        assert t.publish(v).status == Status.ok
        out.append((round(time.perf_counter() - w0, 4), round(t.stats().last_publish_ms, 1)))
    print(json.dumps({"publish_wall_s_device_ms": out}))


if __name__ == "__main__":
    main()
