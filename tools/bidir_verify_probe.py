"""Both-ways NVLink pull with and without chunk verification (diagnostic).

GPUs 0 and 1 pull `--gb` from each other at once through rs_pull_spans
(the fused pull kernel), in three modes: plain copy; copy + own chunk-digest
table; copy + verify against the source's table + own table (what every
chain hop does).  Separates the link's both-ways limit from the cost of the
integrity traffic.  Prints one JSON line.

    python tools/bidir_verify_probe.py [--gb 4]
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import sys
import threading

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch

    from paper_2604_09107_b200 import ros
    from paper_2604_09107_b200._lib import lib
    ap = argparse.ArgumentParser()
    ap.add_argument("--gb", type=float, default=4.0)
    ap.add_argument("--items", type=int, default=16)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    n = int(a.gb * (1 << 30)) // a.items // 4096 * 4096
    total = n * a.items
    d = [torch.device("cuda", 0), torch.device("cuda", 1)]
    src = [torch.empty(total, dtype=torch.uint8, device=x) for x in d]
    dst = [torch.empty(total, dtype=torch.uint8, device=x) for x in d]
    nck = a.items * ((n // 4096 + 31) // 32 * 32)
    dig = [torch.zeros(nck, dtype=torch.int64, device=x) for x in d]   # source tables
    own = [torch.zeros(nck, dtype=torch.int64, device=x) for x in d]   # receiver tables
    lens = np.asarray([n] * a.items, np.uint64)
    for g in (0, 1):
        ros.synth_bf16(src[g], 21 + g)
        torch.cuda.synchronize(d[g])
        sp = np.asarray([src[g].data_ptr() + i * n for i in range(a.items)], np.uint64)
        code, ms = C.c_int(), C.c_float()
        # the source's table: a local hash-only pass over its own bytes
        assert lib.rs_pull_spans(sp.ctypes.data, None, lens.ctypes.data, a.items, 4096, None,
                                 C.c_void_p(dig[g].data_ptr()), g, None, C.byref(code), C.byref(ms)) == 0
        assert code.value == 0

    def run(dirs, mode):
        res = {}
        barrier = threading.Barrier(len(dirs))

        def one(g):  # g pulls from 1-g
            s_ = np.asarray([src[1 - g].data_ptr() + i * n for i in range(a.items)], np.uint64)
            d_ = np.asarray([dst[g].data_ptr() + i * n for i in range(a.items)], np.uint64)
            exp = C.c_void_p(dig[1 - g].data_ptr()) if mode == "verify" else None
            out = C.c_void_p(own[g].data_ptr()) if mode in ("digests", "verify") else None
            code, ms = C.c_int(), C.c_float()
            times = []
            barrier.wait()
            for _ in range(a.reps + 4):
                rc = lib.rs_pull_spans(s_.ctypes.data, d_.ctypes.data, lens.ctypes.data, a.items, 4096,
                                       exp, out, g, None, C.byref(code), C.byref(ms))
                assert rc == 0 and code.value == 0, (rc, code.value)
                times.append(ms.value)
            mid = sorted(times[2:-2])
            res[g] = round(total / (mid[len(mid) // 2] / 1e3) / 1e9, 1)

        ths = [threading.Thread(target=one, args=(g,)) for g in dirs]
        for t in ths:
            t.start()
        for t in ths:
            t.join()
        if mode == "verify":
            for g in dirs:
                assert torch.equal(own[g].cpu(), dig[1 - g].cpu())
        return [res[g] for g in dirs]

    out = {"bytes_per_direction": total, "peer_boxes": os.environ.get("RSB_PEER_BOXES", "")}
    for mode in ("plain", "digests", "verify"):
        out[f"uni_{mode}"] = run([0], mode)
        out[f"bi_{mode}"] = run([0, 1], mode)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
