"""GPU: cross-link seed buffers end to end (reference ClientCore
start_seed_fill / local_step, client_core.cpp:262-302, 1720-1812; ServerCore
seeding, server_core.cpp:915-970, 1124-1204).

A replica in another datacenter opened with offload_seed does not pull a new
version over the cross-datacenter link on update: its update reports no
change and a background fill lands the version in pinned host memory (the
pull kernel writes it over PCIe, verifying every chunk against the source's
table and writing the seed's own).  Same-datacenter readers are then planned
onto the seed, and the owner's next update consumes it locally (copy-engine
frames from host memory, verified in place).  The test mirrors
test_client_core.cpp:460-503."""
import time

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


SIZES = {0: [("w", 200000), ("big", (12 << 20) + 4099)], 1: [("x", 100000), ("y", 5 << 20)]}


def _replica(cl, name, dc, fill, **cfg):
    from paper_2604_09107_b200 import ros
    from paper_2604_09107_b200.ros import Status
    h = cl.open("m", name, 2, datacenter=dc, **cfg)
    bufs = {}
    for shard, ents in SIZES.items():
        for i, (n, size) in enumerate(ents):
            b = torch.zeros(size, dtype=torch.uint8, device="cuda:0")
            if fill:
                ros.synth_bf16(b[: size // 2 * 2], 100 + 10 * shard + i)
            bufs[(shard, n)] = b
            assert h.register_tensor(shard, n, b) == Status.ok
    torch.cuda.synchronize()
    return h, bufs


def _same(a, b):
    return all(torch.equal(a[k], b[k]) for k in a)


TOTAL = sum(s for ents in SIZES.values() for _, s in ents)


def test_cross_link_update_fills_a_host_seed_then_consumes_it_locally():
    from paper_2604_09107_b200.ros import Cluster, Status
    cl = Cluster()
    try:
        t, tb = _replica(cl, "T", "dc1", True)
        assert t.publish(1).status == Status.ok
        f, fb = _replica(cl, "F", "dc2", False, offload_seed=True)
        # first poll: the version is masked for dc2, a background fill starts
        r = f.update("latest")
        assert r.status == Status.ok and not r.changed and r.version is None
        assert f.seed_lanes() == [1]  # waits for the fill
        v = cl.view("m", "F+seed@1")
        assert v["lifecycle"] == "published" and v["kind"] == "offload" and not v["seeding"]
        st = f.stats()
        assert st.bytes_pulled_cross_dc == TOTAL and st.bytes_copied_local == 0
        assert not any(b.any() for b in fb.values())  # F's regions untouched so far
        # a same-datacenter neighbour is planned onto the seed (host memory)
        n, nb = _replica(cl, "N", "dc2", False)
        r = n.replicate("latest")
        assert r.status == Status.ok and r.version == 1
        assert [a.src for a in cl.assigns() if a.replica == "N"] == ["F+seed@1"]
        assert _same(nb, tb)
        # second poll: the change lands by consuming the local seed
        r = f.update("latest")
        assert r.status == Status.ok and r.changed and r.version == 1
        assert f.current_version == 1
        assert _same(fb, tb)
        for s in range(2):
            assert (f.chunk_digests(s) == t.chunk_digests(s)).all()
        st = f.stats()
        assert st.bytes_copied_local == TOTAL
        assert st.bytes_pulled_cross_dc == TOTAL  # only the fill crossed the link
        assert "seed_consumed model=m replica=F" in cl.trace()
        # consumed and drained: the buffer is handed back and the lane vanishes
        f.poll()
        assert cl.view("m", "F+seed@1") is None
        assert f.seed_lanes() == []
    finally:
        cl.close()


def test_failed_seed_fill_is_dropped_and_the_version_stays_masked_until_refilled():
    """A corrupted source: the seed fill's kernel rejects the bytes
    (checksum), the registry voids and releases the seed, and the owner's
    next update starts a fresh fill (the source fixed by then)."""
    from paper_2604_09107_b200.ros import Cluster, Status
    cl = Cluster()
    try:
        t, tb = _replica(cl, "T", "dc1", True)
        assert t.publish(1).status == Status.ok
        good = tb[(0, "big")][7 << 20].item()
        tb[(0, "big")][7 << 20] ^= 0x5A  # corrupt after publish
        torch.cuda.synchronize()
        f, fb = _replica(cl, "F", "dc2", False, offload_seed=True, pull_timeout_s=1.0)
        r = f.update("latest")
        assert r.status == Status.ok and not r.changed
        f.seed_wait()
        assert "replica_voided model=m replica=F+seed@1 reason=seed_failed" in cl.trace()
        f.poll()
        assert f.seed_lanes() == [] and cl.view("m", "F+seed@1") is None
        tb[(0, "big")][7 << 20] = good
        torch.cuda.synchronize()
        r = f.update("latest")
        assert r.status == Status.ok and not r.changed
        assert f.seed_lanes() == [1]
        r = f.update("latest")
        assert r.status == Status.ok and r.changed and r.version == 1
        assert _same(fb, tb)
    finally:
        cl.close()
