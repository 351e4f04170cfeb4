"""Retention offload lanes: RetentionRule
(types.hpp:119-123), unpublish_needs_offload / on_offload_confirm /
create_offload_replica / eval_offload_releases (server_core.cpp:1387-1485,
1592-1645) and the client's retention lane (client_core.cpp:1675-1717).

CPU: the registry's behaviour on the reference's own unit-test scenarios
(tests/unit/test_server_core.cpp:424-510), and the registry trace of a
retention cycle against the reference library driven live (oracle/_ref).
GPU: the lane is pinned host memory; a reader pulls the parked version out
of it through the pull kernel (in-process, and from another process)."""
import ctypes as C
import os
import time
import re
import socket

import numpy as np
import pytest

from paper_2604_09107_b200._lib import lib
from paper_2604_09107_b200.ros import Cluster, Status
from tests.conftest import ROOT
from tests.test_reshard import _open


def _publish(cl, replica, v, man):
    arr = (C.c_char_p * 1)(man)
    lens = (C.c_size_t * 1)(len(man))
    return lib.rs_server_publish(cl.h, b"m", replica.encode(), v, 1, C.cast(arr, C.c_void_p),
                                 C.cast(lens, C.c_void_p), None, None)


def _retain(cl, replica, lags):
    arr = (C.c_uint64 * len(lags))(*lags)
    assert lib.rs_server_set_retention(cl.h, b"m", replica.encode(), C.cast(arr, C.c_void_p),
                                       len(lags)) == 0


def _result(cl, replica):
    d, s, v, ch = C.c_int(), C.c_int(), C.c_uint64(), C.c_int()
    lib.rs_server_result(cl.h, b"m", replica.encode(), C.byref(d), C.byref(s), C.byref(v), C.byref(ch))
    return bool(d.value), s.value, v.value


def _pending(cl, replica):
    v = C.c_uint64()
    return lib.rs_server_offload_pending(cl.h, b"m", replica.encode(), C.byref(v)), v.value


def _manifest(oracle, salt):
    ng, g, off = oracle.assemble([1 << 20])
    return oracle.manifest_encode(["w"], [1 << 20], [salt], g, off, ng, [])


def test_offload_parked_then_released(oracle):
    """test_server_core.cpp:424-474."""
    cl = Cluster()
    _open(cl, "watcher", 1, "")
    _retain(cl, "watcher", [0, 1])
    _open(cl, "trainer", 1, "")
    assert _publish(cl, "trainer", 1, _manifest(oracle, 1)) == 0
    # v1 is retained (lag 0 against max=1) and nothing else holds it
    assert lib.rs_server_unpublish(cl.h, b"m", b"trainer") == 0
    assert _pending(cl, "trainer") == (1, 1)
    assert not _result(cl, "trainer")[0]
    # the client copies v1 to host memory and confirms
    assert lib.rs_server_offload_confirm(cl.h, b"m", b"trainer", 0, 1, 1, b"host:trainer:0") == 0
    assert _result(cl, "trainer")[:2] == (True, 0)
    ov = cl.view("m", "trainer+offload@1")
    assert ov["kind"] == "offload" and ov["version"] == 1 and ov["visible"]
    # next cycle: v2 goes up; v1 (lag 1) stays retained, the offload survives
    assert _publish(cl, "trainer", 2, _manifest(oracle, 2)) == 0
    assert cl.view("m", "trainer+offload@1") is not None
    # a reader replicates v1 out of the offload...
    _open(cl, "reader", 1, "")
    loc = cl.locate("m", "reader", "1")
    assert loc["source_replica"] == "trainer+offload@1"
    assert loc["source_endpoint"] == "host:trainer:0"
    assert lib.rs_server_replicate(cl.h, b"m", b"reader", b"1") == 0
    assert lib.rs_server_complete(cl.h, b"m", b"reader", 0, 0) == 0
    # ...after which a durable worker copy exists and the buffer is released
    assert cl.view("m", "trainer+offload@1") is None
    assert cl.releases("m", "trainer") == [1]
    cl.close()


def test_two_retained_versions_parked_concurrently(oracle):
    """test_server_core.cpp:476-510."""
    cl = Cluster()
    _open(cl, "watcher", 1, "")
    _retain(cl, "watcher", [0, 1])
    _open(cl, "trainer", 1, "")
    for v in (1, 2):
        assert _publish(cl, "trainer", v, _manifest(oracle, v)) == 0
        assert lib.rs_server_unpublish(cl.h, b"m", b"trainer") == 0
        assert _pending(cl, "trainer") == (1, v)
        assert lib.rs_server_offload_confirm(cl.h, b"m", b"trainer", 0, v, 1, b"host:trainer:0") == 0
        assert _result(cl, "trainer")[:2] == (True, 0)
    assert cl.view("m", "trainer+offload@1") is not None
    assert cl.view("m", "trainer+offload@2") is not None
    listing = cl.listing("m")
    assert listing[1] == {"trainer+offload@1"} and listing[2] == {"trainer+offload@2"}
    # v3 shifts the retained window to {3, 2}: v1's buffer goes, v2's stays
    assert _publish(cl, "trainer", 3, _manifest(oracle, 3)) == 0
    assert cl.view("m", "trainer+offload@1") is None
    assert cl.view("m", "trainer+offload@2") is not None
    assert cl.releases("m", "trainer") == [1]
    cl.close()


def test_offload_failure_keeps_the_copy_published(oracle):
    """on_offload_confirm with ok=false (server_core.cpp:1404-1421)."""
    cl = Cluster()
    _open(cl, "watcher", 1, "")
    _retain(cl, "watcher", [0])
    _open(cl, "trainer", 1, "")
    assert _publish(cl, "trainer", 1, _manifest(oracle, 1)) == 0
    assert lib.rs_server_unpublish(cl.h, b"m", b"trainer") == 0
    assert lib.rs_server_offload_confirm(cl.h, b"m", b"trainer", 0, 1, 0, b"") == 0
    assert _result(cl, "trainer")[:2] == (True, int(Status.offload_failed))
    v = cl.view("m", "trainer")
    assert v["lifecycle"] == "published" and v["visible"]
    assert cl.view("m", "trainer+offload@1") is None
    cl.close()


_KEEP = ("publish_commit", "unpublish_start", "offload_first", "offload_confirmed",
         "offload_replica", "unpublish_ack", "replicate_resolved", "assign", "replica_complete",
         "offload_release_start", "offload_released")


def _server_lines(text, ref):
    out = []
    for line in text.splitlines():
        if ref:
            m = re.match(r"^\d+ \d+ A (\S+)(.*)$", line)
        else:
            m = re.match(r"^\d+ (\S+)(.*)$", line)
        if m and m.group(1) in _KEEP:
            out.append((m.group(1) + m.group(2)).strip())
    return out


@pytest.mark.skipif(not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "librefstore_ref.so")),
                    reason="reference library not built")
def test_retention_cycle_matches_reference_library(oracle):
    """The same retention cycle on the reference ServerCore (driven through
    its own ClientCore + MemNetwork) and on our registry: identical server
    events -- offload_first, the offload replica, the reader assigned to it,
    and the release once the reader holds the version."""
    c = oracle.RefCluster(threaded=False)
    for r in ("watcher", "trainer", "reader"):
        c.add(r)
    assert c.set_retention("watcher", [0, 1]) == 0
    assert c.open("watcher") == 0
    a = oracle.synth_bf16(1, 1 << 18).view(np.uint8)
    b, w = np.zeros_like(a), np.zeros_like(a)
    c.register("trainer", 0, "w", a)
    c.register("reader", 0, "w", b)
    c.register("watcher", 0, "w", w)
    assert c.publish("trainer", 1)[0] == 0
    assert c.unpublish("trainer") == 0
    sts, vs, _, _ = c.pull_many(["reader"], spec="1")
    c.settle()
    assert sts == [0] and vs == [1] and np.array_equal(a, b)
    ref = _server_lines(c.trace(), ref=True)
    c.close()

    cl = Cluster()
    man = oracle.publish_manifest(["w"], [a])
    _open(cl, "watcher", 1, "")
    _retain(cl, "watcher", [0, 1])
    _open(cl, "trainer", 1, "")
    assert _publish(cl, "trainer", 1, man) == 0
    assert lib.rs_server_unpublish(cl.h, b"m", b"trainer") == 0
    assert lib.rs_server_offload_confirm(cl.h, b"m", b"trainer", 0, 1, 1, b"ep:trainer") == 0
    _open(cl, "reader", 1, "")
    assert lib.rs_server_replicate(cl.h, b"m", b"reader", b"1") == 0
    assert lib.rs_server_complete(cl.h, b"m", b"reader", 0, 0) == 0
    ours = _server_lines(cl.trace(), ref=False)
    cl.close()
    assert ours == ref, (ours, ref)


# --------------------------------------------------------------------- GPU
torch = pytest.importorskip("torch")


def _need_gpu(n=1):
    if not torch.cuda.is_available() or torch.cuda.device_count() < n:
        pytest.skip(f"needs {n} CUDA device(s)")


def _tensors(dev, seed, sizes=((6 << 20) + 4096 * 3, 5000, 3 << 20)):
    from paper_2604_09107_b200 import ros
    out = []
    for i, n in enumerate(sizes):
        t = torch.empty(n, dtype=torch.uint8, device=dev)
        ros.synth_bf16(t, seed + i)
        out.append(t)
    return out


@pytest.mark.gpu
def test_gpu_reader_pulls_parked_version_from_host():
    """The trainer's unpublish parks v1 in pinned host memory; it then
    publishes new bytes as v2 in place.  A reader asking for v1 is served by
    the offload through the pull kernel (host memory over PCIe), bit-exact;
    once the reader holds v1 the registry releases the buffer."""
    _need_gpu()
    dev = torch.device("cuda:0")
    with Cluster() as cl:
        w = cl.open("m", "watcher", 1)
        wt = torch.zeros(4096, dtype=torch.uint8, device=dev)
        assert w.register_tensor(0, "w0", wt) == Status.ok
        w.set_retention([0, 1])
        assert w.connect() == Status.ok
        t = cl.open("m", "trainer", 1, tiny_threshold=1 << 20)
        tb = _tensors(dev, 10)
        for i, x in enumerate(tb):
            assert t.register_tensor(0, f"w{i}", x) == Status.ok
        assert t.publish(1).status == Status.ok
        v1 = [x.clone() for x in tb]
        d1 = t.chunk_digests(0)
        assert t.unpublish().status == Status.ok
        assert t.lanes() == [1]
        assert cl.view("m", "trainer+offload@1")["kind"] == "offload"
        # new weights in place, published as v2: v1 now lives only in the offload
        for i, x in enumerate(tb):
            from paper_2604_09107_b200 import ros
            ros.synth_bf16(x, 100 + i)
        assert t.publish(2).status == Status.ok
        r = cl.open("m", "reader", 1, tiny_threshold=1 << 20)
        rb = [torch.zeros_like(x) for x in tb]
        for i, x in enumerate(rb):
            assert r.register_tensor(0, f"w{i}", x) == Status.ok
        res = r.replicate("1")
        assert res.status == Status.ok and res.version == 1, res
        assert [(a.replica, a.src) for a in cl.assigns()][-1] == ("reader", "trainer+offload@1")
        torch.cuda.synchronize()
        for a, b in zip(v1, rb):
            assert torch.equal(a, b)
        assert np.array_equal(r.chunk_digests(0), d1)
        # a worker holds v1 again: the offload is released and its buffer freed
        assert cl.view("m", "trainer+offload@1") is None
        t.poll()
        assert t.lanes() == []


@pytest.mark.gpu
def test_corrupted_parked_version_fails_loudly():
    """A byte flipped in the pinned host lane after parking: the copy engine
    lands it, the pull kernel's chunk check catches it (the re-read sees the
    same bad byte), and the replicate fails instead of handing out wrong
    weights."""
    import glob
    import mmap
    _need_gpu()
    dev = torch.device("cuda:0")
    with Cluster() as cl:
        w = cl.open("m", "watcher", 1)
        assert w.register_tensor(0, "w0", torch.zeros(4096, dtype=torch.uint8, device=dev)) == Status.ok
        w.set_retention([0, 1])
        assert w.connect() == Status.ok
        t = cl.open("m", "trainer", 1, tiny_threshold=1 << 20)
        tb = _tensors(dev, 30)
        for i, x in enumerate(tb):
            assert t.register_tensor(0, f"w{i}", x) == Status.ok
        before = set(glob.glob(f"/dev/shm/rsb-{os.getpid()}-*"))
        assert t.publish(1).status == Status.ok
        assert t.unpublish().status == Status.ok
        assert t.lanes() == [1]
        lane = sorted(set(glob.glob(f"/dev/shm/rsb-{os.getpid()}-*")) - before,
                      key=os.path.getsize)[-1]
        with open(lane, "r+b") as f, mmap.mmap(f.fileno(), 0) as mm:
            mm[1 << 20] ^= 0x40  # inside the first item
        from paper_2604_09107_b200 import ros
        for i, x in enumerate(tb):
            ros.synth_bf16(x, 300 + i)
        assert t.publish(2).status == Status.ok
        r = cl.open("m", "reader", 1, tiny_threshold=1 << 20, pull_timeout_s=2.0)
        for i, x in enumerate(tb):
            assert r.register_tensor(0, f"w{i}", torch.zeros_like(x)) == Status.ok
        res = r.replicate("1")
        # the chunk check fails; the failure report condemns the only source
        # of v1 (the reference: item_failed -> failure_report, client_core.cpp:336-357)
        assert res.status in (Status.checksum_mismatch, Status.version_unavailable), res
        assert r.stats().checksum_failures >= 1
        assert not r.is_published


@pytest.mark.gpu
def test_failed_copy_engine_fill_is_drained_before_returning():
    """A corrupted host lane fails the copy-engine fill at its first frame;
    the frames already queued behind it must be drained before the fill's
    outcome is acted on (a retry from another source would otherwise be
    overwritten, and the lane could be released while the engine still
    reads it).  Once replicate has returned, nothing lands any more."""
    import glob
    import mmap
    _need_gpu()
    dev = torch.device("cuda:0")
    from paper_2604_09107_b200 import ros
    sizes = (1 << 30, 5000)
    with Cluster() as cl:
        w = cl.open("m", "watcher", 1)
        assert w.register_tensor(0, "w0", torch.zeros(4096, dtype=torch.uint8, device=dev)) == Status.ok
        w.set_retention([0, 1])
        assert w.connect() == Status.ok
        t = cl.open("m", "trainer", 1, tiny_threshold=1 << 20)
        tb = _tensors(dev, 40, sizes)
        for i, x in enumerate(tb):
            assert t.register_tensor(0, f"w{i}", x) == Status.ok
        before = set(glob.glob(f"/dev/shm/rsb-{os.getpid()}-*"))
        assert t.publish(1).status == Status.ok
        assert t.unpublish().status == Status.ok
        assert t.lanes() == [1]
        lane = sorted(set(glob.glob(f"/dev/shm/rsb-{os.getpid()}-*")) - before,
                      key=os.path.getsize)[-1]
        with open(lane, "r+b") as f, mmap.mmap(f.fileno(), 0) as mm:
            mm[1 << 20] ^= 0x40  # first frame: stops the fill
        for i, x in enumerate(tb):
            ros.synth_bf16(x, 500 + i)
        assert t.publish(2).status == Status.ok
        r = cl.open("m", "reader", 1, tiny_threshold=1 << 20, pull_timeout_s=2.0)
        rb = [torch.zeros_like(x) for x in tb]
        for i, x in enumerate(rb):
            assert r.register_tensor(0, f"w{i}", x) == Status.ok
        res = r.replicate("1")
        assert res.status != Status.ok, res
        assert r.stats().checksum_failures >= 1
        snap = rb[0].clone()
        torch.cuda.synchronize()
        time.sleep(0.1)  # a stray copy-engine frame (128 MiB: ~2.4 ms) would land by now
        assert torch.equal(snap, rb[0])


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _dist_worker(rank, world, port, q):
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
        sizes = [(6 << 20) + 4096 * 3, 5000, 3 << 20]
        if rank == 0:
            w = dc.create("m", "watcher", 1)
            assert w.register_tensor(0, "w0", torch.zeros(4096, dtype=torch.uint8, device=dev)) == 0
            w.set_retention([0, 1])
        dc.open(w if rank == 0 else None)
        bufs = [torch.zeros(n, dtype=torch.uint8, device=dev) for n in sizes]
        h = dc.create("m", "trainer" if rank == 0 else "reader", 1, tiny_threshold=1 << 20)
        for i, b in enumerate(bufs):
            assert h.register_tensor(0, f"w{i}", b) == Status.ok
        dc.open(h)
        if rank == 0:
            for i, b in enumerate(bufs):
                ros.synth_bf16(b, 10 + i)
            torch.cuda.synchronize()
        assert (dc.publish(h if rank == 0 else None, 1) or ros.OpResult(Status.ok)).status == 0
        v1 = dc.gather(ros.digest_spans([b.data_ptr() for b in bufs], sizes, gpu))[0]
        r = dc.unpublish(h if rank == 0 else None)
        out = {"unpublish": None if r is None else int(r.status)}
        if rank == 0:
            out["lanes_after_unpublish"] = h.lanes()
            for i, b in enumerate(bufs):
                ros.synth_bf16(b, 100 + i)
            torch.cuda.synchronize()
        dc.publish(h if rank == 0 else None, 2)
        res = dc.replicate(h if rank == 1 else None, "1")
        if rank == 1:
            out["replicate"] = (int(res.status), res.version)
            out["bytes_v1"] = ros.digest_spans([b.data_ptr() for b in bufs], sizes, gpu) == v1
        out["plan"] = [(a.replica, a.src) for a in dc.assigns()]
        dist.barrier()
        if rank == 0:
            h.poll()
            out["lanes_after_release"] = h.lanes()
        q.put((rank, out))
        dc.close()
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - surfaced by the parent
        import traceback
        q.put((rank, {"error": repr(e) + traceback.format_exc()}))
        raise


@pytest.mark.gpu
def test_gpu_reader_in_another_process_pulls_the_offload():
    """The offload lane is POSIX shared memory registered with CUDA: the
    reader's process maps it by name and its pull kernel reads it (one GPU:
    both processes on cuda:0)."""
    _need_gpu(1)
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_dist_worker, args=(r, 2, port, q)) for r in range(2)]
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
    assert res[0]["unpublish"] == 0 and res[0]["lanes_after_unpublish"] == [1]
    assert res[1]["replicate"] == (0, 1) and res[1]["bytes_v1"]
    assert ("reader", "trainer+offload@1") in res[1]["plan"]
    assert res[0]["lanes_after_release"] == []


@pytest.mark.gpu
def test_early_published_version_parked_and_served_with_its_final_manifest(oracle):
    """An early publish (big-entry digests in the background) that is later
    parked in host memory: the unpublish waits for the digests, the offload
    serves the version, and a reader ends with the reference's manifest."""
    _need_gpu()
    dev = torch.device("cuda:0")
    from paper_2604_09107_b200 import ros
    sizes = ((6 << 20) + 4096 * 3, 5000, 3 << 20)
    with Cluster() as cl:
        w = cl.open("m", "watcher", 1)
        assert w.register_tensor(0, "w0", torch.zeros(4096, dtype=torch.uint8, device=dev)) == Status.ok
        w.set_retention([0, 1])
        assert w.connect() == Status.ok
        t = cl.open("m", "trainer", 1, tiny_threshold=1 << 20, early_publish=True)
        tb = _tensors(dev, 70, sizes)
        for i, x in enumerate(tb):
            assert t.register_tensor(0, f"w{i}", x) == Status.ok
        assert t.publish(1).status == Status.ok
        v1 = [x.clone() for x in tb]
        want = oracle.publish_manifest([f"w{i}" for i in range(3)],
                                       [x.cpu().numpy() for x in v1], tiny=1 << 20)
        assert t.unpublish().status == Status.ok  # waits for the digests, then parks
        assert t.lanes() == [1] and not t.publish_pending
        for i, x in enumerate(tb):
            ros.synth_bf16(x, 170 + i)
        assert t.publish(2).status == Status.ok
        r = cl.open("m", "reader", 1, tiny_threshold=1 << 20)
        rb = [torch.zeros_like(x) for x in tb]
        for i, x in enumerate(rb):
            assert r.register_tensor(0, f"w{i}", x) == Status.ok
        res = r.replicate("1")
        assert res.status == Status.ok and res.version == 1, res
        assert [(a.replica, a.src) for a in cl.assigns()][-1] == ("reader", "trainer+offload@1")
        torch.cuda.synchronize()
        for a, b in zip(v1, rb):
            assert torch.equal(a, b)
        assert r.manifest(0) == want
