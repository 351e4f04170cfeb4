"""GPU: a reader PROCESS that did not exist when the others started joins
through the registry's operation log and chases a copy that is still filling
(config 4's elastic join with dynamic membership; shared.py, oplog.cpp).
The trainer publishes early (rs_config.early_publish): readers pull while its
big-entry digests run, and the final manifest reaches every member through
the log afterwards.

  process 0   hosts the log; trainer T publishes 1 GiB + tiny tensors; reader
              A is planned and bound (serving its empty fill) but not filling
  process 1   joins only now: replays the log, opens reader B, replicates ->
              planned onto A (a pipeline copy, source_complete == 0), imports
              A's serve state (CUDA IPC) from the log, launches and waits on
              A's watermarks; process 0 then fills A and B chases it.

No gloo group, no collective: process 1 is not known to anyone until it
appends its first entry.  With one GPU both processes share cuda:0."""
import os

import pytest

from tests.conftest import ROOT

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

SIZES = [1 << 30, 6000, 3 << 20]


def _bufs(dev, seed=None):
    from paper_2604_09107_b200 import ros
    out = []
    for i, n in enumerate(SIZES):
        b = torch.zeros(n, dtype=torch.uint8, device=dev)
        if seed is not None:
            ros.synth_bf16(b, seed + i)
        out.append(b)
    return out


def _host(q, joined, done):
    import sys
    sys.path.insert(0, ROOT)
    import torch

    from paper_2604_09107_b200 import ros
    from paper_2604_09107_b200.ros import Status
    from paper_2604_09107_b200.shared import LogServer, SharedCluster
    try:
        dev = torch.device("cuda", 0)
        log = LogServer()
        sc = SharedCluster("127.0.0.1", log.port)
        t = sc.create("m", "T", 1, tiny_threshold=1 << 20, early_publish=True)
        tb = _bufs(dev, seed=800)
        for i, b in enumerate(tb):
            assert t.register_tensor(0, f"w{i}", b) == Status.ok
        a = sc.create("m", "A", 1, tiny_threshold=1 << 20, pull_timeout_s=30.0)
        ab = _bufs(dev)
        for i, b in enumerate(ab):
            assert a.register_tensor(0, f"w{i}", b) == Status.ok
        torch.cuda.synchronize()
        sc.open(t)
        sc.open(a)
        assert sc.publish(t, 1).status == Status.ok
        assert sc.replicate_start(a) is None  # bound and serving, nothing landed
        q.put(("host", "port", {"port": log.port}))
        # the joiner is planned onto A while A has not started filling
        import time
        t0 = time.time()
        while time.time() - t0 < 120:
            v = sc.local.view("m", "B")
            if v and v["lifecycle"] == "replicating":
                break
            time.sleep(0.01)
        time.sleep(0.5)  # B binds, imports A's serve state and launches its chase
        res = {"a": sc.replicate_finish(a)}
        joined.wait(120)
        want = ros.digest_spans([b.data_ptr() for b in tb], SIZES, 0)
        got_a = ros.digest_spans([b.data_ptr() for b in ab], SIZES, 0)
        sc.sync()
        q.put(("host", "final", {"a": int(res["a"].status), "a_equal": got_a == want, "want": want,
                                 "t_manifest": t.manifest(0), "a_manifest": a.manifest(0),
                                 "assigns": [(x.replica, x.src) for x in sc.assigns()],
                                 "listing": {v: sorted(r) for v, r in sc.listing("m").items()}}))
        done.wait(120)
        sc.close()
        log.close()
    except Exception as e:  # pragma: no cover - surfaced by the parent
        import traceback
        q.put(("host", "error", repr(e) + traceback.format_exc()))


def _joiner(port, q, joined):
    import sys
    sys.path.insert(0, ROOT)
    import torch

    from paper_2604_09107_b200 import ros
    from paper_2604_09107_b200.ros import Status
    from paper_2604_09107_b200.shared import SharedCluster
    try:
        dev = torch.device("cuda", torch.cuda.device_count() - 1)
        sc = SharedCluster("127.0.0.1", port)
        b = sc.create("m", "B", 1, tiny_threshold=1 << 20, pull_timeout_s=30.0)
        bb = _bufs(dev)
        for i, x in enumerate(bb):
            assert b.register_tensor(0, f"w{i}", x) == Status.ok
        sc.open(b)
        r = sc.replicate(b)
        a = b.transfer_assignment(0)
        got = ros.digest_spans([x.data_ptr() for x in bb], SIZES, dev.index)
        # early publish: the final manifest reaches this member through the log
        q.put(("joiner", "final", {"b": int(r.status), "v": r.version, "assignment": a, "digests": got,
                                   "manifest": b.manifest(0)}))
        joined.set()
        sc.close()
    except Exception as e:  # pragma: no cover - surfaced by the parent
        import traceback
        q.put(("joiner", "error", repr(e) + traceback.format_exc()))
        joined.set()


def test_reader_process_joins_mid_fill_through_the_op_log():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    joined, done = ctx.Event(), ctx.Event()
    host = ctx.Process(target=_host, args=(q, joined, done))
    host.start()
    procs = [host]
    try:
        who, what, info = q.get(timeout=300)
        assert what == "port", info
        j = ctx.Process(target=_joiner, args=(info["port"], q, joined))
        j.start()
        procs.append(j)
        res = {}
        for _ in range(2):
            who, what, r = q.get(timeout=300)
            assert what == "final", r
            res[who] = r
        assert res["host"]["a"] == 0 and res["host"]["a_equal"]
        jb = res["joiner"]
        assert jb["b"] == 0 and jb["v"] == 1, jb
        assert jb["assignment"]["source_replica"] == "A", jb
        assert jb["assignment"]["source_complete"] is False, jb  # chased a filling copy
        assert jb["digests"] == res["host"]["want"]
        assert ("A", "T") in res["host"]["assigns"] and ("B", "A") in res["host"]["assigns"]
        assert res["host"]["listing"] == {1: ["A", "B", "T"]}
        # T published early (big-entry digests in the background): every
        # member ends with the reference's build_publish_payload bytes
        import sys
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import numpy as np
        import oracle as O
        arrs = [O.synth_bf16(800 + i, n // 2) for i, n in enumerate(SIZES)]
        want = O.publish_manifest([f"w{i}" for i in range(len(SIZES))], arrs, tiny=1 << 20)
        assert res["host"]["t_manifest"] == want
        assert res["host"]["a_manifest"] == want
        assert jb["manifest"] == want
    finally:
        done.set()
        joined.set()
        for p in procs:
            p.join(timeout=60)


def _group_member(rank, port, q):
    """Process `rank` of a TP-2 trainer group (trainer shard = rank) that also
    holds shard (rank + 1) % 2 of a TP-2 reader replica; process 0 also holds
    a TP-1 reader that reshards from both trainer shards.  Every replica
    operation is a group transaction through the op log."""
    import hashlib
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import torch

    from paper_2604_09107_b200 import ros
    from paper_2604_09107_b200.ros import Status, tp_slice
    from paper_2604_09107_b200.shared import SharedCluster
    from tests.test_cast import _tensors
    from tests.test_reshard import numel
    try:
        gpu = rank % torch.cuda.device_count()
        torch.cuda.set_device(gpu)
        dev = torch.device("cuda", gpu)
        sc = SharedCluster("127.0.0.1", port)
        tiny = 64 << 10
        tensors = _tensors()
        full = {}
        for i, (n, shape, _) in enumerate(tensors):  # every process builds the same bytes
            t = torch.empty(numel(shape) * 2, dtype=torch.uint8, device=dev)
            ros.synth_bf16(t, 700 + i)
            full[n] = t

        def piece(n, geo):
            rows, w, r0, nr, c0, nc = geo
            return full[n].view(rows, w)[r0:r0 + nr, c0:c0 + nc].contiguous().view(-1)

        t = sc.create("m", "trainer", 2, tiny_threshold=tiny, early_publish=True)
        keep = []
        for n, shape, dim in tensors:
            geo = tp_slice(shape, 2, dim, 2, rank)
            keep.append(piece(n, geo))
            assert t.register_slice(rank, n, keep[-1], geo) == Status.ok
        sc.open(t, endpoints={rank: f"p{rank}:cuda{gpu}"})
        s = (rank + 1) % 2
        r = sc.create("m", "tp2", 2, tiny_threshold=tiny)
        rb = {}
        for n, shape, dim in tensors:
            geo = tp_slice(shape, 2, dim, 2, s)
            rb[n] = torch.zeros(geo[3] * geo[5], dtype=torch.uint8, device=dev)
            assert r.register_slice(s, n, rb[n], geo) == Status.ok
        sc.open(r, endpoints={s: f"p{rank}:cuda{gpu}"})
        out = {"publish": int(sc.publish(t, 1).status)}
        out["tp2"] = int(sc.replicate(r).status)
        if rank == 0:
            u = sc.create("m", "tp1", 1, tiny_threshold=tiny)
            ub = {}
            for n, shape, _ in tensors:
                ub[n] = torch.zeros_like(full[n])
                assert u.register_slice(0, n, ub[n], tp_slice(shape, 2, None, 1, 0)) == Status.ok
            sc.open(u)
            out["tp1"] = int(sc.replicate(u).status)
        torch.cuda.synchronize()
        bad = []
        for n, shape, dim in tensors:
            if not torch.equal(rb[n], piece(n, tp_slice(shape, 2, dim, 2, s))):
                bad.append(("tp2", n))
            if rank == 0 and not torch.equal(ub[n], full[n]):
                bad.append(("tp1", n))
        out["bad"] = bad
        out["t_manifest"] = hashlib.sha256(t.manifest(rank)).hexdigest()  # final bytes (early publish)
        out["r_manifest"] = hashlib.sha256(r.manifest(s)).hexdigest()
        out["plan"] = sorted({(a.replica, a.src) for a in sc.assigns()})
        q.put((rank, out))
        sc.finalized(t)
        import time
        time.sleep(1.0)  # let the other member read what it needs before this one leaves
        sc.close()
    except Exception as e:  # pragma: no cover - surfaced by the parent
        import traceback
        q.put((rank, {"error": repr(e) + traceback.format_exc()}))


def test_tp_group_split_over_processes_via_group_transactions():
    """A TP-2 trainer and a TP-2 reader whose shards live in two processes,
    plus a TP-1 reader resharding from both: open, publish (early) and
    replicate are group transactions in the op log (no gloo, no collective).
    Bytes equal the numpy slices; each reader shard's manifest is the
    trainer shard's final one."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import multiprocessing as mp
    from paper_2604_09107_b200.shared import LogServer
    log = LogServer()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_group_member, args=(r, log.port, q)) for r in range(2)]
    try:
        for p in ps:
            p.start()
        res = dict(q.get(timeout=300) for _ in range(2))
        for r in range(2):
            assert "error" not in res[r], res[r].get("error")
            o = res[r]
            assert o["publish"] == 0 and o["tp2"] == 0, o
            assert o["bad"] == [], o["bad"]
        assert res[0]["tp1"] == 0
        # the reader shard s holds trainer shard s's bytes: the same manifest
        assert res[0]["r_manifest"] == res[1]["t_manifest"]
        assert res[1]["r_manifest"] == res[0]["t_manifest"]
        plan = dict(res[0]["plan"])
        assert plan["tp2"] == "trainer" and plan["tp1"] in ("trainer", "tp2"), plan
    finally:
        for p in ps:
            p.join(timeout=60)
        log.close()


def _retention_member(role, port, q, ev):
    """role 'trainer': hosts nothing but its replica + a retention watcher;
    parks v1 in host memory on unpublish.  role 'reader': joins later and
    pulls v1 from the parked lane (POSIX shm mapped by name) via the log."""
    import sys
    sys.path.insert(0, ROOT)
    import torch

    from paper_2604_09107_b200 import ros
    from paper_2604_09107_b200.ros import Status
    from paper_2604_09107_b200.shared import SharedCluster
    try:
        dev = torch.device("cuda", 0)
        sc = SharedCluster("127.0.0.1", port)
        sizes = [(6 << 20) + 4096 * 3, 5000, 3 << 20]
        if role == "trainer":
            w = sc.create("m", "watcher", 1)
            assert w.register_tensor(0, "w0", torch.zeros(4096, dtype=torch.uint8, device=dev)) == Status.ok
            w.set_retention([0, 1])
            sc.open(w)
            t = sc.create("m", "trainer", 1, tiny_threshold=1 << 20)
            tb = [torch.empty(n, dtype=torch.uint8, device=dev) for n in sizes]
            for i, b in enumerate(tb):
                ros.synth_bf16(b, 910 + i)
                assert t.register_tensor(0, f"w{i}", b) == Status.ok
            torch.cuda.synchronize()
            sc.open(t)
            assert sc.publish(t, 1).status == Status.ok
            v1 = ros.digest_spans([b.data_ptr() for b in tb], sizes, 0)
            r = sc.unpublish(t)
            out = {"unpublish": int(r.status), "lanes": t.lanes(), "v1": v1}
            for i, b in enumerate(tb):
                ros.synth_bf16(b, 1910 + i)
            torch.cuda.synchronize()
            out["publish2"] = int(sc.publish(t, 2).status)
            q.put(("trainer", out))
            ev.wait(120)
            sc.sync()
            q.put(("trainer2", {"view": sc.local.view("m", "trainer+offload@1")}))
        else:
            r = sc.create("m", "reader", 1, tiny_threshold=1 << 20)
            rb = [torch.zeros(n, dtype=torch.uint8, device=dev) for n in sizes]
            for i, b in enumerate(rb):
                assert r.register_tensor(0, f"w{i}", b) == Status.ok
            sc.open(r)
            res = sc.replicate(r, "1")
            q.put(("reader", {"status": int(res.status), "v": res.version,
                              "digests": ros.digest_spans([b.data_ptr() for b in rb], sizes, 0),
                              "plan": [(a.replica, a.src) for a in sc.assigns()]}))
            ev.set()
        sc.close()
    except Exception as e:  # pragma: no cover - surfaced by the parent
        import traceback
        q.put((role, {"error": repr(e) + traceback.format_exc()}))
        ev.set()


def test_retention_offload_through_the_op_log():
    """The last durable copy of a retained version unpublishes: its process
    parks it in pinned host memory (POSIX shm) and announces the lane through
    the log; a reader process that joins afterwards replicates that version
    from the lane (copy-engine frames verified in place by its pull kernel)
    and, once a worker holds it again, the registry releases the offload."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import multiprocessing as mp
    from paper_2604_09107_b200.shared import LogServer
    log = LogServer()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ev = ctx.Event()
    tr = ctx.Process(target=_retention_member, args=("trainer", log.port, q, ev))
    tr.start()
    procs = [tr]
    try:
        who, out = q.get(timeout=300)
        assert who == "trainer" and "error" not in out, out
        assert out["unpublish"] == 0 and out["lanes"] == [1] and out["publish2"] == 0
        rd = ctx.Process(target=_retention_member, args=("reader", log.port, q, ev))
        rd.start()
        procs.append(rd)
        res = dict(q.get(timeout=300) for _ in range(2))
        assert "error" not in res["reader"], res["reader"]
        assert res["reader"]["status"] == 0 and res["reader"]["v"] == 1
        assert res["reader"]["digests"] == out["v1"]
        assert ("reader", "trainer+offload@1") in res["reader"]["plan"]
        assert res["trainer2"]["view"] is None  # released once a worker holds v1
    finally:
        ev.set()
        for p in procs:
            p.join(timeout=60)
        log.close()


def _seed_member(role, port, q, evs):
    """T (dc1) publishes v1; F (dc2, offload_seed) updates -> background seed
    fill into host memory, reported through the log; N (dc2, another
    process) is planned onto F's seed and pulls it from F's host lane; F's
    next update consumes its seed locally; the registry then releases it."""
    import sys
    sys.path.insert(0, ROOT)
    import torch

    from paper_2604_09107_b200 import ros
    from paper_2604_09107_b200.ros import Status
    from paper_2604_09107_b200.shared import SharedCluster
    try:
        dev = torch.device("cuda", 0)
        sc = SharedCluster("127.0.0.1", port)
        sizes = [(6 << 20) + 4096 * 3, 5000, 3 << 20]
        bufs = [torch.zeros(n, dtype=torch.uint8, device=dev) for n in sizes]
        dc = "dc1" if role == "T" else "dc2"
        h = sc.create("m", role, 1, tiny_threshold=1 << 20, offload_seed=(role == "F"))
        if role == "T":
            for i, b in enumerate(bufs):
                ros.synth_bf16(b, 710 + i)
        for i, b in enumerate(bufs):
            assert h.register_tensor(0, f"w{i}", b) == Status.ok
        torch.cuda.synchronize()
        sc.open(h, datacenter=dc)
        digests = lambda: ros.digest_spans([b.data_ptr() for b in bufs], sizes, 0)  # noqa: E731
        out = {}
        if role == "T":
            assert sc.publish(h, 1).status == Status.ok
            q.put(("T", {"v1": digests()}))
            evs["done"].wait(300)
        elif role == "F":
            evs["published"].wait(120)
            r = sc.update(h)
            out["first"] = (int(r.status), r.changed)
            sc.seed_wait(h)
            v = sc.local.view("m", "F+seed@1")
            out["seed_view"] = v and (v["lifecycle"], v["kind"])
            out["untouched"] = not any(b.any() for b in bufs)
            q.put(("F1", out))
            evs["neighbour_done"].wait(300)
            r = sc.update(h)
            out = {"second": (int(r.status), r.changed, r.version), "digests": digests(),
                   "src": [(a.replica, a.src) for a in sc.assigns() if a.replica == "F"]}
            sc.sync()
            h.poll()
            out["after_view"] = sc.local.view("m", "F+seed@1")
            out["lanes"] = h.seed_lanes()
            q.put(("F2", out))
        else:  # N
            evs["seeded"].wait(300)
            r = sc.replicate(h)
            q.put(("N", {"status": int(r.status), "v": r.version, "digests": digests(),
                         "src": [(a.replica, a.src) for a in sc.assigns() if a.replica == "N"]}))
            evs["done"].wait(300)
        sc.close()
    except Exception as e:  # pragma: no cover - surfaced by the parent
        import traceback
        q.put((role, {"error": repr(e) + traceback.format_exc()}))


def test_cross_link_seed_through_the_op_log():
    """Seed buffers across processes (client_core.cpp:1720-1812 with the
    op log as the control plane): the seed fill is started by F's update,
    reported with role seed through the log, its host lane announced; a
    same-datacenter reader in a third process pulls the seed; F consumes it
    locally; every byte equals the trainer's."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import multiprocessing as mp
    from paper_2604_09107_b200.shared import LogServer
    log = LogServer()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    evs = {k: ctx.Event() for k in ("published", "seeded", "neighbour_done", "done")}
    procs = [ctx.Process(target=_seed_member, args=(r, log.port, q, evs)) for r in ("T", "F", "N")]
    try:
        for p in procs:
            p.start()
        got = {}
        who, out = q.get(timeout=300)
        assert who == "T" and "error" not in out, out
        got["T"] = out
        evs["published"].set()
        who, out = q.get(timeout=300)
        assert who == "F1" and "error" not in out, (who, out)
        assert out["first"] == (0, False)
        assert out["seed_view"] == ("published", "offload") and out["untouched"]
        evs["seeded"].set()
        who, out = q.get(timeout=300)
        assert who == "N" and "error" not in out, (who, out)
        assert out["status"] == 0 and out["v"] == 1 and out["src"] == [("N", "F+seed@1")]
        assert out["digests"] == got["T"]["v1"]
        evs["neighbour_done"].set()
        who, out = q.get(timeout=300)
        assert who == "F2" and "error" not in out, (who, out)
        assert out["second"] == (0, True, 1)
        assert out["src"] == [("F", "F+seed@1")]
        assert out["digests"] == got["T"]["v1"]
        assert out["after_view"] is None and out["lanes"] == []
    finally:
        evs["done"].set()
        for p in procs:
            p.join(timeout=60)
        log.close()
