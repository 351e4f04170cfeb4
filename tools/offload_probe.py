"""Retention offload probe (diagnostic): park a version in pinned host
memory (the unpublish's offload lane, D2H over PCIe) and pull it back into a
reader through the pull kernel reading host memory.

    python tools/offload_probe.py [--workload llama3_8b]
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
    ap.add_argument("--workload", default="llama3_8b")
    a = ap.parse_args()
    shapes = B.workload_shapes(a.workload)
    total = sum(2 * B._numel(s) for _, s in shapes)
    dev = torch.device("cuda:0")
    ta, tv = B.alloc_replica(shapes, dev, seed_base=42)
    ra, rv = B.alloc_replica(shapes, dev)
    cl = Cluster()
    w = cl.open("m", "watcher", 1)
    wt = torch.zeros(4096, dtype=torch.uint8, device=dev)
    w.register_tensor(0, "w0", wt)
    w.set_retention([0, 1])
    assert w.connect() == Status.ok
    t = cl.open("m", "trainer", 1)
    r = cl.open("m", "reader", 1)
    for (n, v), (_, x) in zip(tv, rv):
        t.register_tensor(0, n, v)
        r.register_tensor(0, n, x)
    assert t.publish(1).status == Status.ok
    t0 = time.perf_counter()
    assert t.unpublish().status == Status.ok  # offload first
    off_s = time.perf_counter() - t0
    t.publish(2)
    res = r.replicate("1")
    assert res.status == Status.ok, res
    st = r.stats()
    torch.cuda.synchronize()
    ok = torch.equal(ta, ra)
    # second cycle: v1 is released (a worker holds it) and its pinned buffer
    # is reused for parking v2
    t.poll()
    t1 = time.perf_counter()
    assert t.unpublish().status == Status.ok
    off2_s = time.perf_counter() - t1
    print(json.dumps({"workload": a.workload, "bytes": total, "offload_s": round(off_s, 4),
                      "offload_gbs": round(total / off_s / 1e9, 2),
                      "offload_reused_s": round(off2_s, 4),
                      "offload_reused_gbs": round(total / off2_s / 1e9, 2),
                      "pull_from_host_ms": round(st.last_pull_ms, 3),
                      "pull_from_host_gbs": round(total / (st.last_pull_ms / 1e3) / 1e9, 2),
                      "bytes_equal": ok, "plan": [(x.replica, x.src) for x in cl.assigns()]}))
    cl.close()


if __name__ == "__main__":
    main()
