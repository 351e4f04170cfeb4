"""Off-box data plane (transport_stream.hpp:36-76):
serve states over TCP.  A source advertised as "tcp:<host>:<port>" is pulled
through the process's stream server: the reader receives the chunk map,
digest table and payload batches into pinned host memory and its pull
kernel lands and verifies them, chasing the per-batch host watermarks.

GPU, loopback: bytes and chunk digests equal the source's; a second reader
chained behind the first chases it over the wire; a source that goes away
mid-stream fails the fill loudly."""
import threading

import numpy as np
import pytest

from paper_2604_09107_b200.ros import Cluster, Status

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(autouse=True)
def need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _bufs(dev, seed=None, sizes=((48 << 20) + 4096 * 5 + 100, 7000, 3 << 20)):
    from paper_2604_09107_b200 import ros
    out = []
    for i, n in enumerate(sizes):
        t = torch.zeros(n, dtype=torch.uint8, device=dev)
        if seed is not None:
            ros.synth_bf16(t[: n // 2 * 2], seed + i)
        out.append(t)
    return out


def _open(cl, name, bufs, ep=None):
    h = cl.open("m", name, 1, tiny_threshold=1 << 20)
    for i, b in enumerate(bufs):
        assert h.register_tensor(0, f"w{i}", b) == Status.ok
    if ep:
        h.set_endpoint(0, ep)
    return h


def test_pull_over_tcp_is_bit_exact():
    dev = torch.device("cuda:0")
    with Cluster() as cl:
        port = cl.listen()
        ep = f"tcp:127.0.0.1:{port}"
        tb = _bufs(dev, seed=5)
        t = _open(cl, "trainer", tb, ep)
        assert t.publish(1).status == Status.ok
        rb = _bufs(dev)
        r = _open(cl, "reader", rb, ep)
        res = r.replicate()
        assert res.status == Status.ok, res
        torch.cuda.synchronize()
        for a, b in zip(tb, rb):
            assert torch.equal(a, b)
        assert np.array_equal(r.chunk_digests(0), t.chunk_digests(0))


def test_chained_readers_chase_each_other_over_tcp():
    """r1 chases r0 while r0 is still landing -- across the wire.  The two
    readers sit on different GPUs: persistent pull kernels that wait on each
    other must not share one GPU (a chaser could occupy every SM first)."""
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    with Cluster() as cl:
        port = cl.listen()
        ep = f"tcp:127.0.0.1:{port}"
        tb = _bufs(torch.device("cuda:0"), seed=9)
        t = _open(cl, "trainer", tb, ep)
        assert t.publish(1).status == Status.ok
        devs = [torch.device("cuda:1"), torch.device("cuda:0")]
        readers = [(_open(cl, f"r{i}", rb, ep), rb) for i, rb in
                   enumerate([_bufs(d) for d in devs])]
        results = {}

        def run(h):
            results[h.replica] = h.replicate()

        ths = [threading.Thread(target=run, args=(h,)) for h, _ in readers]
        for th in ths:
            th.start()
        for th in ths:
            th.join()
        assert all(v.status == Status.ok for v in results.values()), (results, cl.trace()[-3000:])
        srcs = [a.src for a in cl.assigns()]
        assert len(set(srcs)) == len(srcs)  # a chain: every copy serves one reader
        for d in devs:
            torch.cuda.synchronize(d)
        for _, rb in readers:
            for a, b in zip(tb, rb):
                assert torch.equal(a.cpu(), b.cpu())


def test_unreachable_tcp_source_fails_loudly():
    dev = torch.device("cuda:0")
    with Cluster() as cl:
        tb = _bufs(dev, seed=3)
        t = _open(cl, "trainer", tb, "tcp:127.0.0.1:9")  # nothing listens there
        assert t.publish(1).status == Status.ok
        r = _open(cl, "reader", _bufs(dev))
        res = r.replicate(wait_s=20.0)
        assert res.status != Status.ok


def test_version_bumps_over_tcp_reuse_pinned_buffers():
    """Consecutive versions land through the same (pooled) pinned buffers:
    every version's bytes are exact, none served stale."""
    from paper_2604_09107_b200 import ros
    dev = torch.device("cuda:0")
    with Cluster() as cl:
        port = cl.listen()
        ep = f"tcp:127.0.0.1:{port}"
        tb = _bufs(dev, seed=21)
        t = _open(cl, "trainer", tb, ep)
        rb = _bufs(dev)
        r = _open(cl, "reader", rb, ep)
        for v in range(1, 5):
            if v > 1:
                assert t.unpublish().status == Status.ok
                for i, x in enumerate(tb):
                    ros.synth_bf16(x[: x.numel() // 2 * 2], 1000 * v + i)
                torch.cuda.synchronize()
            assert t.publish(v).status == Status.ok
            res = r.update() if v > 1 else r.replicate()
            assert res.status == Status.ok and res.version == v, res
            torch.cuda.synchronize()
            for a, b in zip(tb, rb):
                assert torch.equal(a, b), v
