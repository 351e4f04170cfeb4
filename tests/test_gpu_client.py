"""GPU: the ROS API end to end through the C ABI, mirroring the reference's
ClusterFix scenarios (tests/unit/test_client_core.cpp) with device-resident
regions.  Bytes, manifests, chunk digests and plans are checked against the
CPU oracle / reference fixtures."""
import json
import threading

import numpy as np
import pytest

from tests.conftest import golden
from tests.golden.models import tiny_set

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def pattern(n, salt):
    # fill_pattern of test_client_core.cpp:76-81
    return ((salt * 1315423911 + np.arange(n, dtype=np.uint64) * 131) & 0xFF).astype(np.uint8)


class Fix:
    """ClusterFix with device buffers."""

    def __init__(self, dev=0, **cluster_kw):
        from paper_2604_09107_b200.ros import Cluster
        self.cl = Cluster(**cluster_kw)
        self.h = {}
        self.bufs = {}
        self.dev = dev

    def make(self, replica, shards=1, dev=None, **cfg):
        self.h[replica] = self.cl.open("m", replica, shards, **cfg)
        self.h[replica].devnum = self.dev if dev is None else dev
        return self.h[replica]

    def reg(self, replica, shard, name, n, salt):
        dev = torch.device("cuda", self.h[replica].devnum)
        t = torch.from_numpy(pattern(n, salt)).to(dev)
        self.bufs[(replica, shard, name)] = t
        from paper_2604_09107_b200.ros import Status
        assert self.h[replica].register_tensor(shard, name, t) == Status.ok

    def same(self, a, b, shard, name):
        return torch.equal(self.bufs[(a, shard, name)].cpu(), self.bufs[(b, shard, name)].cpu())

    def close(self):
        self.cl.close()


@pytest.fixture
def fx():
    f = Fix()
    yield f
    f.close()


def test_publish_list_unpublish_roundtrip(fx):
    from paper_2604_09107_b200.ros import Status
    t = fx.make("T", 2)
    fx.reg("T", 0, "a", 3000, 1)
    fx.reg("T", 0, "b", 5000, 2)
    fx.reg("T", 1, "c", 4096, 3)
    r = t.publish(1)
    assert r.status == Status.ok and r.version == 1
    assert t.is_published and t.current_version == 1
    assert fx.cl.listing("m") == {1: {"T"}}
    assert t.unpublish().status == Status.ok
    assert not t.is_published and t.current_version == 1
    assert fx.cl.listing("m") == {}


def test_replicate_pulls_bytes_that_verify(fx, oracle):
    # test_client_core.cpp:163-202
    from paper_2604_09107_b200.ros import Status
    t = fx.make("T", 2)
    for args in [(0, "big", 3 << 20, 7), (0, "t1", 1000, 8), (0, "t2", 2000, 9), (1, "u1", 4096, 10)]:
        fx.reg("T", *args)
    assert t.publish(1).status == Status.ok
    w = fx.make("R", 2)
    for args in [(0, "big", 3 << 20, 100), (0, "t1", 1000, 100), (0, "t2", 2000, 100),
                 (1, "u1", 4096, 100)]:
        fx.reg("R", *args)
    r = w.replicate("latest")
    assert r.status == Status.ok and r.version == 1
    assert w.is_published and w.current_version == 1
    for s, n in [(0, "big"), (0, "t1"), (0, "t2"), (1, "u1")]:
        assert fx.same("T", "R", s, n)
    st = w.stats()
    assert st.items_verified == 3
    assert st.bytes_pulled == (3 << 20) + 1000 + 2000 + 4096
    assert st.checksum_failures == 0
    v = fx.cl.view("m", "R")
    assert v["lifecycle"] == "published" and v["version"] == 1
    # manifests are byte-identical to build_publish_payload's (oracle port,
    # itself pinned to the reference on CPU)
    m0 = oracle.publish_manifest(["big", "t1", "t2"], [pattern(3 << 20, 7), pattern(1000, 8),
                                                         pattern(2000, 9)])
    assert t.manifest(0) == m0 and w.manifest(0) == m0
    assert t.manifest(1) == oracle.publish_manifest(["u1"], [pattern(4096, 10)])
    # chunk digest tables agree with the oracle on both sides
    want0 = oracle.chunk_digests([pattern(3 << 20, 7), np.concatenate([pattern(1000, 8),
                                                                        pattern(2000, 9)])], 4096)
    assert np.array_equal(t.chunk_digests(0), want0)
    assert np.array_equal(w.chunk_digests(0), want0)


def test_manifest_matches_reference_fixture(fx):
    from paper_2604_09107_b200.ros import Status
    m = json.load(open(golden("manifests.json")))
    names, arrays = tiny_set()
    for key, kw in (("tiny_set_real", {}),
                    ("tiny_set_real_small_limits", {"tiny_threshold": 100 << 10,
                                                    "group_target": 1 << 20})):
        h = fx.cl.open("m", "P" + key, 1, **kw)
        keep = []
        for n, a in zip(names, arrays):
            t = torch.from_numpy(a).cuda()
            keep.append(t)
            assert h.register_tensor(0, n, t) == Status.ok
        assert h.publish(1).status == Status.ok
        assert h.manifest(0).hex() == m[key]["encoded"]
        h.unpublish()


def test_chain_of_readers_matches_reference_plan(fx):
    from paper_2604_09107_b200.ros import Status
    plan = json.load(open(golden("plans.json")))["chain7"]
    names = ["trainer"] + [f"rollout{i}" for i in range(1, 8)]
    for i, r in enumerate(names):
        fx.make(r)
        for n, l in plan["tensors"]:
            fx.reg(r, 0, n, l, 1 if r == "trainer" else 50 + i)
    assert fx.h["trainer"].publish(1).status == Status.ok
    # one GPU: run the fills one after another (each upstream completes before
    # its reader launches; chasing across GPUs is covered by the multi-GPU test)
    for r in names[1:]:
        assert fx.h[r].replicate().status == Status.ok
    got = [(a.replica, a.version, a.src, a.src_serving) for a in fx.cl.assigns()]
    want = [(a["replica"], a["version"], a["src"], a["src_serving"]) for a in plan["assigns"]]
    assert got == want
    for r in names[1:]:
        for n, _ in plan["tensors"]:
            assert fx.same("trainer", r, 0, n)


def test_corrupt_source_quiet_retry_report_repick(fx):
    # test_client_core.cpp:346-377
    from paper_2604_09107_b200.ros import Status
    t1 = fx.make("T1")
    fx.reg("T1", 0, "big", 3 << 20, 11)
    fx.reg("T1", 0, "tiny", 5000, 12)
    assert t1.publish(1).status == Status.ok
    t2 = fx.make("T2")
    fx.reg("T2", 0, "big", 3 << 20, 20)
    fx.reg("T2", 0, "tiny", 5000, 21)
    assert t2.replicate().status == Status.ok
    fx.bufs[("T2", 0, "big")][17] ^= 0xFF  # corrupt T2's copy in place
    w = fx.make("R")
    fx.reg("R", 0, "big", 3 << 20, 30)
    fx.reg("R", 0, "tiny", 5000, 31)
    r = w.replicate()
    assert r.status == Status.ok
    st = w.stats()
    assert st.checksum_failures == 2  # first attempt + quiet retry
    assert st.failure_reports == 1
    assert fx.same("T1", "R", 0, "big") and fx.same("T1", "R", 0, "tiny")
    assert "T2" in fx.cl.listing("m")[1]  # corruption does not condemn


def test_silent_source_is_reported_and_pull_moves(fx):
    # test_client_core.cpp:317-344
    from paper_2604_09107_b200.ros import Status
    t1 = fx.make("T1", pull_timeout_s=0.5)
    fx.reg("T1", 0, "w", 150000, 6)
    assert t1.publish(1).status == Status.ok
    t2 = fx.make("T2", pull_timeout_s=0.5)
    fx.reg("T2", 0, "w", 150000, 60)
    assert t2.replicate().status == Status.ok
    fx.cl.set_silent("m", "T2", True)
    w = fx.make("R", pull_timeout_s=0.5)
    fx.reg("R", 0, "w", 150000, 70)
    r = w.replicate()
    assert r.status == Status.ok
    assert w.stats().failure_reports >= 1
    assert fx.same("T1", "R", 0, "w")
    lm = fx.cl.listing("m")
    assert "T2" not in lm[1] and "T1" in lm[1]


def test_update_moves_to_newer_version(fx, oracle):
    from paper_2604_09107_b200.ros import Status
    t = fx.make("T")
    fx.reg("T", 0, "w", 200000, 1)
    assert t.publish(1).status == Status.ok
    w = fx.make("R")
    fx.reg("R", 0, "w", 200000, 2)
    r = w.update("latest")
    assert r.status == Status.ok and r.changed and r.version == 1
    r = w.update("latest")
    assert r.status == Status.ok and not r.changed
    # trainer mutates in place and publishes v2
    assert t.unpublish().status == Status.ok
    fx.bufs[("T", 0, "w")].copy_(torch.from_numpy(pattern(200000, 9)).cuda())
    assert t.publish(2).status == Status.ok
    r = w.update("latest")
    assert r.status == Status.ok and r.changed and r.version == 2
    assert fx.same("T", "R", 0, "w")
    assert w.current_version == 2


def test_resume_moves_no_bytes_then_invalidate_repulls(fx):
    from paper_2604_09107_b200.ros import Status
    t = fx.make("T")
    fx.reg("T", 0, "w", 1 << 20, 1)
    assert t.publish(1).status == Status.ok
    w = fx.make("R")
    fx.reg("R", 0, "w", 1 << 20, 2)
    assert w.replicate().status == Status.ok
    pulled = w.stats().bytes_pulled
    assert w.unpublish().status == Status.ok
    assert w.replicate().status == Status.ok
    assert w.stats().bytes_pulled == pulled  # verified prefix kept: resumed
    assert w.unpublish().status == Status.ok
    w.invalidate()
    assert w.replicate().status == Status.ok
    assert w.stats().bytes_pulled == 2 * pulled


def test_bind_rejects_mismatched_registration(fx):
    from paper_2604_09107_b200.ros import Status
    t = fx.make("T")
    fx.reg("T", 0, "w", 4096, 1)
    assert t.publish(1).status == Status.ok
    w = fx.make("R")
    fx.reg("R", 0, "w", 4000, 2)  # wrong length (client_core.cpp:1601-1608)
    assert w.replicate().status == Status.invalid_argument


def test_multi_gpu_chain_with_chasing():
    """Readers on different GPUs fill concurrently, each chasing its upstream's
    device watermark over NVLink (peer access).  On a one-GPU box three
    readers share cuda:0 with their grids capped to 48 SMs each, so their
    persistent kernels co-reside and chase each other in HBM."""
    n = torch.cuda.device_count()
    from paper_2604_09107_b200.ros import Status
    f = Fix()
    try:
        readers = n - 1 if n > 1 else 3
        cap = {} if n > 1 else {"grid_sms": 48}
        names = ["trainer"] + [f"r{i}" for i in range(1, readers + 1)]
        size = 256 << 20
        for i, r in enumerate(names):
            f.make(r, dev=i % n, **(cap if i else {}))
            f.reg(r, 0, "w", size, 1 if i == 0 else 99)
            f.reg(r, 0, "norm", 8192, 2 if i == 0 else 98)
        assert f.h["trainer"].publish(1).status == Status.ok
        results = {}

        def run(r):
            results[r] = f.h[r].replicate()

        ths = [threading.Thread(target=run, args=(r,)) for r in names[1:]]
        for th in ths:
            th.start()
        for th in ths:
            th.join()
        assert all(v.status == Status.ok for v in results.values()), results
        # threads arrive in any order; the plan is still a chain: every
        # replica serves exactly one downstream reader
        srcs = [a.src for a in f.cl.assigns()]
        assert len(set(srcs)) == len(srcs) and "trainer" in srcs
        for r in names[1:]:
            assert f.same("trainer", r, 0, "w") and f.same("trainer", r, 0, "norm")
            # the fill's source: the trainer or the reader ahead of it in the
            # chain, complete or (a pipeline copy) still filling
            a = f.h[r].transfer_assignment(0)
            assert a["source_replica"] in names and a["source_replica"] != r
    finally:
        f.close()


def test_survey_abi_names_pull_serve_state(fx):
    """rs_pull (= replicate) and rs_serve_state (the device tables a caller
    chains on) from SURVEY.md §8b's recommended boundary."""
    import ctypes as C
    from paper_2604_09107_b200._lib import lib
    from paper_2604_09107_b200.ros import Status
    fx.make("t")
    fx.reg("t", 0, "w", (3 << 20) + 123, 5)
    assert fx.h["t"].publish(1).status == Status.ok
    fx.make("r")
    fx.reg("r", 0, "w", (3 << 20) + 123, 0)
    v = C.c_uint64()
    assert lib.rs_pull(fx.h["r"].h, b"latest", C.c_double(30.0), C.byref(v)) == 0 and v.value == 1
    assert fx.same("t", "r", 0, "w")
    d, f = C.c_void_p(), C.c_void_p()
    ep, nb = C.c_uint32(), C.c_uint32()
    assert lib.rs_serve_state(fx.h["r"].h, 0, C.byref(d), C.byref(f), C.byref(ep), C.byref(nb)) == 0
    assert d.value and f.value and ep.value > 0
    n_chunks = ((3 << 20) + 123 + 4095) // 4096
    assert nb.value == (n_chunks + 31) // 32


def test_measured_topology_reaches_the_planner(fx):
    """The box's NVLink state (NVML) as the planner's topology term: a
    square matrix, 0 on the diagonal, 1 for NVLink/NVSwitch pairs; on such a
    uniform box the chain plan is unchanged."""
    from paper_2604_09107_b200 import ros
    from paper_2604_09107_b200.ros import Status
    m = ros.nvlink_cost_matrix()
    n = len(m)
    assert n == torch.cuda.device_count() and all(len(r) == n for r in m)
    assert all(m[i][i] == 0 for i in range(n)) and all(x in (0, 1, 2) for r in m for x in r)
    names = ["T", "r1", "r2"]
    for i, r in enumerate(names):
        fx.make(r, dev=i % n)
        fx.h[r].set_endpoint(0, f"gpu{i % n}:{r}")
        fx.reg(r, 0, "w", 1 << 20, 5 if i == 0 else 0)
    fx.cl.set_topology([f"gpu{i % n}:{r}" for i, r in enumerate(names)],
                       [[m[i % n][j % n] for j in range(3)] for i in range(3)])
    assert fx.h["T"].publish(1).status == Status.ok
    for r in names[1:]:
        assert fx.h[r].replicate().status == Status.ok
        assert fx.same("T", r, 0, "w")


def test_early_publish_commits_the_reference_manifest_later(oracle):
    """rs_config.early_publish: publish() returns once the chunk-digest table
    and the manifest structure are in (readers bind and pull, verifying chunk
    by chunk); the big entries' XXH64 digests -- a serial chain per entry --
    finish in the background and the committed manifest is then the
    reference's build_publish_payload bytes exactly."""
    import time
    from paper_2604_09107_b200.ros import Cluster, Status
    dev = torch.device("cuda:0")
    names = ["big", "mid", "t1", "t2"]
    host = [oracle.synth_bf16(60 + i, n) for i, n in enumerate([1 << 29, 3 << 20, 3000, 777])]
    with Cluster() as cl:
        t = cl.open("m", "T", 1, early_publish=True)
        r = cl.open("m", "R", 1)
        keep = []
        for n, a in zip(names, host):
            src = torch.from_numpy(a.view(np.int16).copy()).to(dev)
            dst = torch.zeros_like(src)
            keep += [src, dst]
            assert t.register_tensor(0, n, src) == Status.ok
            assert r.register_tensor(0, n, dst) == Status.ok
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        assert t.publish(1).status == Status.ok
        publish_s = time.perf_counter() - t0
        assert t.publish_pending  # the 1 GiB entry's chain (~0.4 s) is still running
        res = r.replicate("latest")
        assert res.status == Status.ok and res.version == 1
        torch.cuda.synchronize()
        for a, d in zip(host, keep[1::2]):
            assert np.array_equal(d.cpu().numpy().view(np.uint16), a)
        want = oracle.publish_manifest(names, host)
        assert r.manifest(0) == want  # waits for the final bytes
        assert t.manifest(0) == want and not t.publish_pending
        assert "manifest_final" in cl.trace()
        # publish returned while the chain was still running (publish_pending
        # above); its wall time is ~3 ms alone but is not asserted: another
        # process's work on a shared box can stretch a host call
        del publish_s
        # a reader arriving afterwards is assigned the final bytes directly
        r2 = cl.open("m", "R2", 1)
        k2 = [torch.zeros_like(x) for x in keep[0::2]]
        for n, x in zip(names, k2):
            assert r2.register_tensor(0, n, x) == Status.ok
        assert r2.replicate("latest").status == Status.ok
        assert r2.manifest(0) == want
        # the next version: unpublish waits for nothing left, new bytes, early again
        assert t.unpublish().status == Status.ok
        from paper_2604_09107_b200 import ros
        ros.synth_bf16(keep[0], 999)
        torch.cuda.synchronize()
        assert t.publish(2).status == Status.ok
        assert r.update("latest").status == Status.ok
        h2 = [keep[0].cpu().numpy().view(np.uint16)] + host[1:]
        assert r.manifest(0) == oracle.publish_manifest(names, h2)
        assert torch.equal(keep[0], keep[1])


def test_ragged_sizes_and_registration_errors(fx, oracle):
    """Sizes around every boundary the path has -- the 16-byte vector, the
    128-byte TMA box column, the 4096-byte chunk, the 32-chunk watermark
    batch and the 2 MiB tiny threshold -- publish and pull bit-exact, with
    the reference's manifest and chunk table.  Registration errors follow
    ClientCore::register_tensor (client_core.cpp:534-553)."""
    from paper_2604_09107_b200.ros import Status
    sizes = [1, 15, 16, 17, 127, 128, 129, 4095, 4096, 4097, 32 * 4096 - 1, 32 * 4096 + 1,
             (2 << 20) - 1, 2 << 20, (2 << 20) + 1, (5 << 20) + 333]
    t = fx.make("T")
    r = fx.make("R")
    names = [f"e{i}" for i in range(len(sizes))]
    for i, (n, size) in enumerate(zip(names, sizes)):
        fx.reg("T", 0, n, size, 40 + i)
        fx.reg("R", 0, n, size, 0)
    # the reference's registration rules
    z = torch.zeros(4, dtype=torch.uint8, device="cuda:0")
    assert t.register_tensor(0, "zero", ptr=z.data_ptr(), nbytes=0) == Status.invalid_argument
    assert t.register_tensor(0, "e0", z) == Status.already_exists
    assert t.register_tensor(0, "bad|name", z) == Status.invalid_argument
    assert t.register_tensor(5, "x", z) == Status.invalid_argument
    assert t.publish(1).status == Status.ok
    assert r.replicate().status == Status.ok
    arrays = [pattern(size, 40 + i) for i, size in enumerate(sizes)]
    want = oracle.publish_manifest(names, arrays)
    assert t.manifest(0) == want and r.manifest(0) == want
    for n in names:
        assert fx.same("T", "R", 0, n), n
    # chunk table over the items in manifest order: big entries, then the
    # packed group (members at their offsets) where its first member sits
    ng, g, off = oracle.assemble(sizes)
    items, seen = [], set()
    for i, a in enumerate(arrays):
        if g[i] < 0:
            items.append(a)
        elif g[i] not in seen:
            seen.add(g[i])
            items.append(np.concatenate([arrays[j] for j in range(len(arrays)) if g[j] == g[i]]))
    assert np.array_equal(r.chunk_digests(0), oracle.chunk_digests(items, 4096))
    assert r.stats().items_verified == len(items)
