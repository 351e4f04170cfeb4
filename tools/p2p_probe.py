"""Single-process NVLink pull probe (diagnostic, not the bench contract).

Trainer replica on cuda:1, reader on cuda:0, complete source (no chasing):
times the pull kernel through the ROS API, plus a torch peer copy of the
same bytes for reference.  Run variants with RSB_TMA_VARIANT / RSB_NO_MAPS /
RSB_PULL_KERNEL.

    python tools/p2p_probe.py [--gb 4] [--items 16]
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
    from paper_2604_09107_b200.ros import Cluster, Status
    ap = argparse.ArgumentParser()
    ap.add_argument("--gb", type=float, default=4.0)
    ap.add_argument("--items", type=int, default=16)
    ap.add_argument("--reps", type=int, default=4)
    ap.add_argument("--src", type=int, default=1)
    ap.add_argument("--dst", type=int, default=0)
    a = ap.parse_args()
    n = int(a.gb * (1 << 30)) // a.items // 4096 * 4096
    sd, dd = torch.device("cuda", a.src), torch.device("cuda", a.dst)
    src = torch.empty(n * a.items, dtype=torch.uint8, device=sd)
    dst = torch.empty(n * a.items, dtype=torch.uint8, device=dd)
    for i in range(a.items):
        ros.synth_bf16(src[i * n:(i + 1) * n], 7 + i)
    torch.cuda.synchronize(sd)
    out = {"env": {k: os.environ.get(k) for k in ("RSB_TMA_VARIANT", "RSB_NO_MAPS", "RSB_PULL_KERNEL")},
           "bytes": n * a.items}
    # torch peer copy baseline
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.device(dd):
        dst.copy_(src)
        torch.cuda.synchronize(dd)
        e0.record()
        for _ in range(a.reps):
            dst.copy_(src)
        e1.record()
        torch.cuda.synchronize(dd)
    out["torch_peer_copy_gbs"] = round(n * a.items * a.reps / (e0.elapsed_time(e1) / 1e3) / 1e9, 1)
    cl = Cluster()
    t = cl.open("m", "trainer", 1)
    r = cl.open("m", "reader", 1)
    for i in range(a.items):
        assert t.register_tensor(0, f"w{i}", src[i * n:(i + 1) * n]) == Status.ok
        assert r.register_tensor(0, f"w{i}", dst[i * n:(i + 1) * n]) == Status.ok
    assert t.publish(1).status == Status.ok
    times = []
    for k in range(a.reps + 1):
        if r.is_published:
            r.unpublish()
        r.invalidate()
        res = r.replicate()
        assert res.status == Status.ok, res
        if k:
            times.append(r.stats().last_pull_ms)
    best = min(times)
    out["pull_ms_best"] = round(best, 3)
    out["pull_gbs"] = round(n * a.items / (best / 1e3) / 1e9, 1)
    out["pull_gbs_mean"] = round(n * a.items / (sum(times) / len(times) / 1e3) / 1e9, 1)
    assert torch.equal(src.to(dd), dst)
    cl.close()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
