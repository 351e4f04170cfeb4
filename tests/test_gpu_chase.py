"""GPU, one device: a reader chasing a source that is still filling.

The reference serves a replicating copy to readers downstream (pipeline
copies, server_core.cpp:1534-1540); a reader pulls only the source's verified
prefix (`compute_slice`, transport.cpp:32-49; `safe_end_locked`,
transport.hpp:66-68) and long-polls for more (client_core.cpp:231-260).  Here
the downstream kernel waits on the upstream's device watermarks instead.  On
one GPU two persistent pull kernels co-reside when their grids are capped
(rs_config.grid_sms), so the whole chase runs on the driver's 1-GPU box:

  T (published) -> A (filling, launched last) -> B (launched first, chasing)

Split phase: B is planned onto A while A is bound but not yet launched, so B's
assignment is a pipeline copy (source_complete == 0) and B's kernel spins on
A's watermarks until A's kernel lands and verifies each batch.  Also: a
silent upstream times B out; an upstream whose fill aborts (corrupt source)
turns B's chase into not_serving."""
import time

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

GRID = 64  # SMs per fill: two fills co-reside on the 148 SMs of a B200


@pytest.fixture(scope="module", autouse=True)
def need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _setup(oracle, sizes=(96 << 20, 8192, 3000), **cfg):
    from paper_2604_09107_b200.ros import Cluster, Status
    cl = Cluster()
    dev = torch.device("cuda", 0)
    names = [f"w{i}" for i in range(len(sizes))]
    host = [oracle.synth_bf16(900 + i, n // 2) for i, n in enumerate(sizes)]
    hs, bufs = {}, {}
    for rep in ("T", "A", "B"):
        kw = dict(cfg)
        if rep != "T":
            kw["grid_sms"] = GRID
        hs[rep] = cl.open("m", rep, 1, **kw)
        for n, a in zip(names, host):
            t = (torch.from_numpy(a.view(np.int16).copy()).to(dev) if rep == "T"
                 else torch.zeros(a.size, dtype=torch.int16, device=dev))
            bufs[(rep, n)] = t
            assert hs[rep].register_tensor(0, n, t) == Status.ok
    assert hs["T"].publish(1).status == Status.ok
    return cl, hs, bufs, names, host


def _plan_ab(hs):
    """A then B planned and bound (serving their empty fills); nothing launched."""
    from paper_2604_09107_b200.ros import Status
    for rep in ("A", "B"):
        assert hs[rep].connect() == Status.ok
        r = hs[rep].server_replicate("latest")
        assert r.status == Status.ok and r.version == 1, (rep, r)
        assert hs[rep].transfer_bind(1) == Status.ok


def test_chaser_follows_a_filling_source_on_one_gpu(oracle):
    from paper_2604_09107_b200.ros import Status
    cl, hs, bufs, names, host = _setup(oracle)
    try:
        _plan_ab(hs)
        # B launches first: its source A is bound, serving, and not filling yet
        assert hs["B"].transfer_launch() == Status.ok
        a = hs["B"].transfer_assignment(0)
        assert a["source_replica"] == "A" and a["source_complete"] is False, a
        time.sleep(0.3)
        done, nb = hs["B"].transfer_progress(0)
        assert nb > 0 and done == 0, (done, nb)  # B is waiting on A's watermarks
        # now the upstream fills; B lands each batch as A verifies it
        assert hs["A"].transfer_launch() == Status.ok
        assert hs["A"].transfer_assignment(0)["source_replica"] == "T"
        assert hs["A"].transfer_assignment(0)["source_complete"] is True
        assert hs["A"].transfer_wait() == [(Status.ok, 0)]
        assert hs["B"].transfer_wait() == [(Status.ok, 0)]
        hs["A"].transfer_finish(1, True)
        hs["B"].transfer_finish(1, True)
        torch.cuda.synchronize()
        for n, a_ in zip(names, host):
            for rep in ("A", "B"):
                assert np.array_equal(bufs[(rep, n)].cpu().numpy().view(np.uint16), a_), (rep, n)
        want = oracle.chunk_digests([host[0], np.concatenate([host[1], host[2]]).view(np.uint16)], 4096)
        for rep in ("T", "A", "B"):
            assert np.array_equal(hs[rep].chunk_digests(0), want), rep
        assert hs["B"].manifest(0) == oracle.publish_manifest(names, host)
        assert cl.view("m", "B")["lifecycle"] == "published"
        # the plan is the reference chain: B's source is A, A's is T
        assert {(x.replica, x.src) for x in cl.assigns()} == {("A", "T"), ("B", "A")}
    finally:
        cl.close()


def test_silent_upstream_times_the_chaser_out(oracle):
    from paper_2604_09107_b200.ros import Status
    cl, hs, bufs, names, host = _setup(oracle, pull_timeout_s=0.5)
    try:
        _plan_ab(hs)
        assert hs["B"].transfer_launch() == Status.ok
        assert hs["B"].transfer_assignment(0)["source_complete"] is False
        t0 = time.time()
        res = hs["B"].transfer_wait()  # A never fills
        assert res[0][0] == Status.timeout, res
        assert time.time() - t0 < 30
        assert hs["B"].transfer_progress(0)[0] == 0
    finally:
        cl.close()


def test_aborted_upstream_is_not_serving(oracle):
    from paper_2604_09107_b200.ros import Status
    cl, hs, bufs, names, host = _setup(oracle, pull_timeout_s=2.0)
    try:
        bufs[("T", "w0")][3] ^= 0x5A  # corrupt the published copy: A's batch 0 fails twice
        _plan_ab(hs)
        assert hs["B"].transfer_launch() == Status.ok
        assert hs["B"].transfer_assignment(0)["source_complete"] is False
        time.sleep(0.1)
        assert hs["A"].transfer_launch() == Status.ok
        ra = hs["A"].transfer_wait()
        rb = hs["B"].transfer_wait()
        assert ra[0] == (Status.checksum_mismatch, 1), ra
        assert rb[0][0] == Status.not_serving, rb
        assert hs["A"].stats().checksum_failures >= 2  # first attempt + the quiet re-pull
    finally:
        cl.close()


def test_registry_sees_item_progress_while_a_fill_lands(oracle):
    """task_progress (client_core.cpp:1414-1439): a fill reports its
    verified item prefix while it runs, so the registry's view of a
    replicating replica advances before completion.  A fill capped to one SM
    lands 16 x 64 MiB slowly enough to watch."""
    from paper_2604_09107_b200.ros import Cluster, Status
    cl = Cluster()
    try:
        dev = torch.device("cuda", 0)
        n, size = 16, 64 << 20
        t = cl.open("m", "T", 1)
        a = cl.open("m", "A", 1, grid_sms=1)
        keep = []
        for i in range(n):
            src = torch.empty(size, dtype=torch.uint8, device=dev)
            from paper_2604_09107_b200 import ros
            ros.synth_bf16(src, 50 + i)
            dst = torch.zeros_like(src)
            keep += [src, dst]
            assert t.register_tensor(0, f"w{i}", src) == Status.ok
            assert a.register_tensor(0, f"w{i}", dst) == Status.ok
        assert t.publish(1).status == Status.ok
        assert a.connect() == Status.ok
        assert a.server_replicate("latest").status == Status.ok
        assert a.transfer_bind(1) == Status.ok
        assert cl.progress("m", "A") == 0
        assert a.transfer_launch() == Status.ok
        seen = set()
        t0 = time.time()
        while time.time() - t0 < 30:
            done, nb = a.transfer_progress(0)  # reads the watermarks, reports the item prefix
            seen.add(cl.progress("m", "A"))
            if done == nb:
                break
        assert a.transfer_wait() == [(Status.ok, 0)]
        mid = sorted(x for x in seen if 0 < x < n)
        assert mid, sorted(seen)  # the view advanced while the fill ran
        a.transfer_finish(1, True)
        assert cl.view("m", "A")["lifecycle"] == "published"
        for i in range(n):
            assert torch.equal(keep[2 * i], keep[2 * i + 1])
    finally:
        cl.close()
