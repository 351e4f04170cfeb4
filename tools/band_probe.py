"""Column-band vs row-block reshard pull on one GPU (diagnostic).

A TP-1 trainer publishes `--tensors` tensors of [rows x cols] bf16; a TP-2
reader on the same GPU takes them split along dim 0 (each shard a contiguous
row block: 2-D tensor-map boxes) or dim 1 (each shard a column band of every
row: 3-D boxes over [rows][q][chunk]).  Prints each shard's pull-kernel time
and its HBM fraction (read + write of the shard's bytes).
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
    ap.add_argument("--tensors", type=int, default=16)
    ap.add_argument("--rows", type=int, default=8192)
    ap.add_argument("--cols", type=int, default=8192)
    ap.add_argument("--dim", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--chunk", type=int, default=4096)
    ap.add_argument("--src-dev", type=int, default=0, help="trainer GPU (reader: cuda:0)")
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    sdev = torch.device("cuda", a.src_dev)
    shape = (a.rows, a.cols)
    nbytes = a.rows * a.cols * 2
    cl = Cluster()
    t = cl.open("m", "trainer", 1, chunk_bytes=a.chunk)
    r = cl.open("m", "tp2", 2, chunk_bytes=a.chunk)
    keep = []
    for i in range(a.tensors):
        w = torch.randint(0, 256, (nbytes,), dtype=torch.uint8, device=sdev)
        keep.append(w)
        assert t.register_slice(0, f"w{i}", w, tp_slice(shape, 2, None, 1, 0)) == Status.ok
        for s in range(2):
            g = tp_slice(shape, 2, a.dim, 2, s)
            buf = torch.empty(g[3] * g[5], dtype=torch.uint8, device=dev)
            keep.append(buf)
            assert r.register_slice(s, f"w{i}", buf, g) == Status.ok
    stream = torch.cuda.Stream(device=dev)
    for s in range(2):
        r.set_stream(s, stream)
    assert t.publish(1).status == Status.ok
    ms = []
    for k in range(a.steps + 2):
        if r.is_published:
            assert r.unpublish().status == Status.ok
        r.invalidate()
        res = r.replicate("latest")
        assert res.status == Status.ok, res
        if k >= 2:
            ms.append(r.stats().fill_sum_ms / 2)
    per_shard = a.tensors * nbytes // 2
    kms = sum(ms) / len(ms)
    hbm = B.measured_peaks()["hbm_gbs"]
    gbs = 2 * per_shard / (kms / 1e3) / 1e9
    print(json.dumps({"src_dev": a.src_dev, "dim": a.dim, "rows": a.rows, "cols": a.cols, "tensors": a.tensors,
                      "chunk": a.chunk, "kernel_ms": round(kms, 3), "hbm_gbs": round(gbs, 1),
                      "ingress_gbs": round(per_shard / (kms / 1e3) / 1e9, 1),
                      "frac": round(gbs / hbm, 4)}))


if __name__ == "__main__":
    main()
