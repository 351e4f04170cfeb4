"""GPU, one process per GPU (gloo for the registry, CUDA IPC for the data):
replicas whose shards live in different processes.

World 2.  A TP-2 trainer holds shard r on GPU r.  Three readers pull it:
  * "tp2": the same slicing, shard s on GPU (s+1) % 2 -- item-for-item pulls
    across NVLink, chunk digests equal to the trainer's;
  * "fp8": the same slicing landed as e4m3 (config 5 in miniature);
  * "tp1": one process holding whole tensors -- a reshard gathering from both
    trainer shards (one local, one over NVLink).
Bytes are checked against the numpy slices of the synthetic tensors and the
oracle cast; the plan against the planner's rules.  With one GPU both
processes share cuda:0 (the serve states still cross processes as CUDA IPC
handles, opened by the other process on the same device)."""
import os
import socket

import numpy as np
import pytest

from tests.conftest import ROOT

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import hashlib
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    import torch
    import torch.distributed as dist

    import oracle as O
    from paper_2604_09107_b200 import ros
    from paper_2604_09107_b200.dist import DistCluster
    from paper_2604_09107_b200.ros import Status, tp_slice
    from tests.test_cast import _tensors
    from tests.test_reshard import numel
    try:
        gpu = rank % torch.cuda.device_count()  # one GPU: both processes share cuda:0
        torch.cuda.set_device(gpu)
        dev = torch.device("cuda", gpu)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        dc = DistCluster()
        tiny = 64 << 10
        tensors = _tensors()
        full = {}
        for i, (n, shape, _) in enumerate(tensors):  # every rank builds the same bytes
            t = torch.empty(numel(shape) * 2, dtype=torch.uint8, device=dev)
            ros.synth_bf16(t, 500 + i)
            full[n] = t

        def piece(n, geo):
            rows, w, r0, nr, c0, nc = geo
            return full[n].view(rows, w)[r0:r0 + nr, c0:c0 + nc].contiguous().view(-1)

        t = dc.create("m", "trainer", 2, tiny_threshold=tiny)
        keep = []
        for n, shape, dim in tensors:
            geo = tp_slice(shape, 2, dim, 2, rank)
            keep.append(piece(n, geo))
            assert t.register_slice(rank, n, keep[-1], geo) == Status.ok
        dc.open(t, endpoints=[f"rank{rank}:cuda{gpu}"])
        s = (rank + 1) % 2  # the reader shard this GPU holds
        r = dc.create("m", "tp2", 2, tiny_threshold=tiny)
        f = dc.create("m", "fp8", 2, tiny_threshold=tiny)
        rb, fb = {}, {}
        for n, shape, dim in tensors:
            geo = tp_slice(shape, 2, dim, 2, s)
            rb[n] = torch.zeros(geo[3] * geo[5], dtype=torch.uint8, device=dev)
            fb[n] = torch.zeros(geo[3] * geo[5] // 2, dtype=torch.uint8, device=dev)
            assert r.register_slice(s, n, rb[n], geo) == Status.ok
            assert f.register_cast(s, n, fb[n], geo[3] * geo[5], geo) == Status.ok
        dc.open(r, endpoints=[f"rank{rank}:cuda{gpu}"])
        dc.open(f, endpoints=[f"rank{rank}:cuda{gpu}"])
        u, ub = None, {}
        if rank == 0:
            u = dc.create("m", "tp1", 1, tiny_threshold=tiny)
            for n, shape, _ in tensors:
                ub[n] = torch.zeros_like(full[n])
                assert u.register_slice(0, n, ub[n], tp_slice(shape, 2, None, 1, 0)) == Status.ok
        dc.open(u)
        out = {}
        out["publish"] = int(dc.publish(t, 1).status)
        out["tp2"] = int(dc.replicate(r).status)
        out["fp8"] = int(dc.replicate(f).status)
        res_u = dc.replicate(u)
        if rank == 0:
            out["tp1"] = int(res_u.status)
        torch.cuda.synchronize()
        bad = []
        for n, shape, dim in tensors:
            geo = tp_slice(shape, 2, dim, 2, s)
            want = piece(n, geo)
            if not torch.equal(rb[n], want):
                bad.append(("tp2", n))
            cast = torch.empty_like(fb[n])
            ros.bf16_to_e4m3(want, cast)
            torch.cuda.synchronize()
            if not torch.equal(fb[n], cast):
                bad.append(("fp8", n))
            if rank == 0 and not torch.equal(ub[n], full[n]):
                bad.append(("tp1", n))
        # the oracle's cast on the host for a few tensors
        for n, shape, dim in tensors[-3:]:
            geo = tp_slice(shape, 2, dim, 2, s)
            host = piece(n, geo).cpu().numpy().view(np.uint16)
            if not np.array_equal(fb[n].cpu().numpy(), O.bf16_to_e4m3(host)):
                bad.append(("fp8-oracle", n))
        out["bad"] = bad
        dig = lambda h, sh: hashlib.sha256(h.chunk_digests(sh).tobytes()).hexdigest()
        hs = dc.gather({"t": dig(t, rank), "r": dig(r, s), "f": dig(f, s)})
        out["digests_equal"] = hs[rank]["r"] == hs[s]["t"] and hs[rank]["f"] == hs[s]["t"]
        out["plan"] = sorted({(a.replica, a.src) for a in dc.assigns()})
        q.put((rank, out))
        dc.close()
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - surfaced by the parent
        import traceback
        q.put((rank, {"error": repr(e) + traceback.format_exc()}))
        raise


def test_replicas_split_across_processes():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = {}
    for _ in range(2):
        r = q.get(timeout=300)
        res[r[0]] = r[1]
    for p in ps:
        p.join(timeout=60)
    for r in range(2):
        assert "error" not in res[r], res[r].get("error")
        o = res[r]
        assert o["publish"] == 0 and o["tp2"] == 0 and o["fp8"] == 0, o
        assert o["bad"] == [], o["bad"]
        assert o["digests_equal"]
        plan = dict(o["plan"])
        # tp2 comes from the trainer; the later readers from any complete copy
        # that is not terminal (the planner prefers the least recently used)
        assert plan["tp2"] == "trainer" and plan["fp8"] in ("trainer", "tp2"), plan
        assert plan["tp1"] in ("trainer", "tp2"), plan
    assert res[0]["tp1"] == 0


def _bump_worker(rank, world, port, q):
    """Trainer (rank 0) re-publishes new bytes 4 times; the reader (rank 1)
    updates each time through the split-phase calls (launch, poll, wait)."""
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    import torch
    import torch.distributed as dist

    from paper_2604_09107_b200 import ros
    from paper_2604_09107_b200.dist import DistCluster
    from paper_2604_09107_b200.ros import Status
    try:
        gpu = rank % torch.cuda.device_count()  # one GPU: both processes share cuda:0
        torch.cuda.set_device(gpu)
        dev = torch.device("cuda", gpu)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        dc = DistCluster()
        sizes = [(64 << 20) + 4096 * 7, 3000, 5 << 20]
        bufs = [torch.zeros(n, dtype=torch.uint8, device=dev) for n in sizes]
        name = "trainer" if rank == 0 else "reader"
        h = dc.create("m", name, 1, tiny_threshold=1 << 20)
        for i, b in enumerate(bufs):
            assert h.register_tensor(0, f"w{i}", b) == Status.ok
        dc.open(h)
        out, seen = [], []
        for v in range(1, 5):
            r = dc.unpublish(h if (rank == 0 and v > 1) else None)
            if r is not None:
                assert r.status == Status.ok
            if rank == 0:
                for i, b in enumerate(bufs):
                    ros.synth_bf16(b, 100 * v + i)
                torch.cuda.synchronize()
                assert dc.publish(h, v).status == Status.ok
                dc.replicate_start(None)
                res = dc.replicate_finish(None)
            else:
                dc.publish(None, v)
                dc.replicate_start(h, "latest", update=v > 1)
                done, nb = dc.progress(h, 0)
                seen.append((done, nb))
                res = dc.replicate_finish(h)
                out.append((int(res.status), res.version))
            digest = ros.digest_spans([b.data_ptr() for b in bufs], sizes, gpu)
            got = dc.gather(digest)
            out.append(got[0] == got[1])
        q.put((rank, {"out": out, "seen": seen}))
        dc.close()
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - surfaced by the parent
        import traceback
        q.put((rank, {"error": repr(e) + traceback.format_exc()}))
        raise


def test_version_bumps_across_processes():
    """Regression: a re-published owner frees and re-allocates its tables; the
    reader's process must drop its stale IPC mappings (failed on the third
    version before).  Bytes equal after every bump."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_bump_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = {}
    for _ in range(2):
        r = q.get(timeout=300)
        res[r[0]] = r[1]
    for p in ps:
        p.join(timeout=60)
    for r in range(2):
        assert "error" not in res[r], res[r].get("error")
    assert res[0]["out"] == [True] * 4
    reader = res[1]["out"]
    assert reader == [(0, 1), True, (0, 2), True, (0, 3), True, (0, 4), True], reader
    assert all(nb > 0 for _, nb in res[1]["seen"])


def _join_worker(rank, world, port, q):
    """Rank 0: the trainer T and a reader A whose fill is slowed to one SM;
    rank 1: a late joiner B, planned while A is part-way through its fill.
    B's assignment is A as a pipeline copy (source_complete == 0) and B's
    kernel -- in another process, on the IPC-imported serve state -- chases
    A's watermarks (config 4's elastic join; server_core.cpp:1534-1540)."""
    import sys
    import time
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    import torch
    import torch.distributed as dist

    from paper_2604_09107_b200 import ros
    from paper_2604_09107_b200.dist import DistCluster
    from paper_2604_09107_b200.ros import Status
    try:
        gpu = rank % torch.cuda.device_count()
        torch.cuda.set_device(gpu)
        dev = torch.device("cuda", gpu)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        dc = DistCluster()
        sizes = [1 << 30, 6000, 3 << 20]

        def make(name, seed=None, **cfg):
            h = dc.create("m", name, 1, tiny_threshold=1 << 20, pull_timeout_s=30.0, **cfg)
            bufs = [torch.zeros(n, dtype=torch.uint8, device=dev) for n in sizes]
            for i, b in enumerate(bufs):
                if seed is not None:
                    ros.synth_bf16(b, seed + i)
                assert h.register_tensor(0, f"w{i}", b) == Status.ok
            return h, bufs

        if rank == 0:
            t, tb = make("T", seed=700)
            a, ab = make("A", grid_sms=1)
            torch.cuda.synchronize()
        else:
            b, bb = make("B")
        dc.open(t if rank == 0 else b, endpoints=[f"rank{rank}:cuda{gpu}"])
        dc.open(a if rank == 0 else None, endpoints=[f"rank{rank}:cuda{gpu}"])
        assert (dc.publish(t if rank == 0 else None, 1) or ros.OpResult(Status.ok)).status == 0
        out = {}
        dc.replicate_start(a if rank == 0 else None, "latest")
        if rank == 0:
            t0 = time.time()
            while True:
                done, nb = dc.progress(a, 0)
                if done > 0 or time.time() - t0 > 20:
                    break
                time.sleep(1e-4)
            out["a_progress_at_join"] = (done, nb)
        dist.barrier(group=dc.pg)
        dc.replicate_start(b if rank == 1 else None, "latest")
        if rank == 1:
            out["b_assignment"] = b.transfer_assignment(0)
        res = dc.replicate_finish(a if rank == 0 else b)
        out["status"] = int(res.status)
        mine = tb if rank == 0 else bb
        dig = ros.digest_spans([x.data_ptr() for x in mine], sizes, gpu)
        if rank == 0:
            out["a_equal"] = ros.digest_spans([x.data_ptr() for x in ab], sizes, gpu) == dig
        got = dc.gather(dig)
        out["b_equal"] = got[0] == got[1]
        out["tables"] = dc.gather(__import__("hashlib").sha256(
            (a if rank == 0 else b).chunk_digests(0).tobytes()).hexdigest())
        out["plan"] = sorted({(x.replica, x.src) for x in dc.assigns()})
        q.put((rank, out))
        dc.close()
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - surfaced by the parent
        import traceback
        q.put((rank, {"error": repr(e) + traceback.format_exc()}))
        raise


def test_late_joiner_in_another_process_chases_a_filling_copy():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_join_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = {}
    for _ in range(2):
        r = q.get(timeout=300)
        res[r[0]] = r[1]
    for p in ps:
        p.join(timeout=60)
    for r in range(2):
        assert "error" not in res[r], res[r].get("error")
        assert res[r]["status"] == 0, res[r]
        assert res[r]["b_equal"]
    done, nb = res[0]["a_progress_at_join"]
    assert 0 < done < nb, (done, nb)  # A was part-way through when B was planned
    a = res[1]["b_assignment"]
    assert a["source_replica"] == "A" and a["source_complete"] is False, a
    assert res[0]["a_equal"]
    assert res[0]["tables"][0] == res[0]["tables"][1]  # A's and B's chunk tables
    assert ("A", "T") in res[0]["plan"] and ("B", "A") in res[0]["plan"]
