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


def _open(cl, name, bufs, ep=None, **cfg):
    h = cl.open("m", name, 1, tiny_threshold=1 << 20, **cfg)
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
    """r1 chases r0 while r0 is still landing -- across the wire.  With two
    GPUs the readers sit on different GPUs; on one GPU their persistent pull
    kernels wait on each other, so each is capped to 64 SMs (rs_config
    grid_sms) and the two co-reside."""
    n = torch.cuda.device_count()
    cap = {} if n > 1 else {"grid_sms": 64}
    with Cluster() as cl:
        port = cl.listen()
        ep = f"tcp:127.0.0.1:{port}"
        tb = _bufs(torch.device("cuda:0"), seed=9)
        t = _open(cl, "trainer", tb, ep)
        assert t.publish(1).status == Status.ok
        devs = [torch.device("cuda", 1 % n), torch.device("cuda:0")]
        readers = [(_open(cl, f"r{i}", rb, ep, **cap), rb) for i, rb in
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


def _hostile_server(reply):
    """A TCP peer speaking the stream handshake (stream.cpp serve_conn) that
    answers every request with `reply(sock, stripe)`."""
    import socket
    import struct
    ls = socket.socket()
    ls.bind(("127.0.0.1", 0))
    ls.listen(16)
    stop = threading.Event()

    def recv_n(c, n):
        b = b""
        while len(b) < n:
            k = c.recv(n - len(b))
            if not k:
                raise ConnectionError
            b += k
        return b

    def serve():
        ls.settimeout(0.2)
        while not stop.is_set():
            try:
                c, _ = ls.accept()
            except OSError:
                continue
            try:
                _magic, klen = struct.unpack("<II", recv_n(c, 8))
                recv_n(c, klen)
                _version, stripe, _streams = struct.unpack("<QII", recv_n(c, 16))
                c.sendall(struct.pack("<I", 0))
                reply(c, stripe)
            except (ConnectionError, OSError):
                pass
            threading.Timer(5.0, c.close).start()

    th = threading.Thread(target=serve, daemon=True)
    th.start()
    return ls.getsockname()[1], stop


def _vec(fmt, xs):
    import struct
    return struct.pack("<I", len(xs)) + struct.pack("<%d%s" % (len(xs), fmt), *xs)


@pytest.mark.parametrize("case", ["bad_header", "oversized_frame"])
def test_hostile_tcp_source_is_rejected(case):
    """A peer whose header disagrees with itself, or whose frame claims more
    bytes than its batches hold, fails the fill (protocol error) instead of
    writing past the reader's pinned landing buffer."""
    import struct
    n = 1 << 20  # one item: 256 chunks of 4096 B, one batch row of 8

    def reply(c, stripe):
        if stripe != 0:
            return
        count = [n // 4096 + (1 if case == "bad_header" else 0)]
        # chunk0, chunk_len, count, item lengths, member-cut runs (none), digests
        c.sendall(_vec("I", [0, 256]) + _vec("I", [4096]) + _vec("I", count) + _vec("Q", [n]) +
                  _vec("I", [0]) + _vec("Q", []) + _vec("Q", [0] * 256))
        if case == "oversized_frame":
            c.sendall(struct.pack("<IIQ", 0, 1, 1 << 30) + b"\0" * 4096)

    port, stop = _hostile_server(reply)
    dev = torch.device("cuda:0")
    try:
        with Cluster() as cl:
            t = _open(cl, "trainer", [torch.ones(n, dtype=torch.uint8, device=dev)],
                      f"tcp:127.0.0.1:{port}")
            assert t.publish(1).status == Status.ok
            r = cl.open("m", "reader", 1, tiny_threshold=1 << 20, pull_timeout_s=1.0)
            rb = torch.zeros(n, dtype=torch.uint8, device=dev)
            assert r.register_tensor(0, "w0", rb) == Status.ok
            res = r.replicate(wait_s=20.0)
            assert res.status != Status.ok, res
            assert not r.is_published
            assert int(rb.sum()) == 0  # nothing landed from the hostile peer
    finally:
        stop.set()


def test_reference_wire_frozen_request_is_served():
    """The B200 TCP server answers the reference data wire (RSDP,
    transport_stream.hpp:36-76).  The request is the reference's frozen
    byte vector (test_transport.cpp:91-131: header "RSDP" v1 pull_req, body
    model "m", replica "R", version 7, shard 2, offset 4096, max_bytes
    8 MiB); the response is parsed by the same layout and must carry the
    stream bytes [4096, 4096 + 8 MiB) of replica R's shard 2."""
    import socket
    import struct
    dev = torch.device("cuda:0")
    with Cluster() as cl:
        port = cl.listen()
        h = cl.open("m", "R", 3, tiny_threshold=1 << 20)
        bufs = []
        for s in range(3):
            b = torch.zeros(16 << 20, dtype=torch.uint8, device=dev)
            from paper_2604_09107_b200 import ros
            ros.synth_bf16(b, 70 + s)
            bufs.append(b)
            assert h.register_tensor(s, f"w{s}", b) == Status.ok
        assert h.publish(7).status == Status.ok
        req = bytes.fromhex("525344500001" "0001" "0000000000000036"
                            "0102" "00000001" "6d" "0202" "00000001" "52"
                            "0301" "0000000000000007" "0401" "0000000000000002"
                            "0501" "0000000000001000" "0601" "0000000000800000")
        c = socket.create_connection(("127.0.0.1", port))
        c.sendall(req)

        def recv_n(n):
            out = b""
            while len(out) < n:
                k = c.recv(n - len(out))
                assert k, "connection closed"
                out += k
            return out

        magic, ver, kind, blen = struct.unpack(">IHHQ", recv_n(16))
        assert (magic, ver, kind) == (0x52534450, 1, 2) and blen == 18 + (8 << 20)
        st, prog, comp, plen = struct.unpack(">BQBQ", recv_n(18))
        assert (st, prog, comp, plen) == (0, 1, 1, 8 << 20)
        payload = recv_n(plen)
        assert payload == bufs[2][4096:4096 + (8 << 20)].cpu().numpy().tobytes()
        # query_req (test_transport.cpp:146-168 layout): min_items 1 -> complete
        body = (b"\x01\x02" + struct.pack(">I", 1) + b"m" + b"\x02\x02" + struct.pack(">I", 1) + b"R" +
                b"\x03\x01" + struct.pack(">Q", 7) + b"\x04\x01" + struct.pack(">Q", 2) +
                b"\x05\x01" + struct.pack(">Q", 1))
        c.sendall(struct.pack(">IHHQ", 0x52534450, 1, 3, len(body)) + body)
        magic, ver, kind, blen = struct.unpack(">IHHQ", recv_n(16))
        assert (kind, blen) == (4, 10)
        assert struct.unpack(">BQB", recv_n(10)) == (0, 1, 1)
        c.close()


def test_reference_wire_serves_only_the_verified_prefix_of_a_filling_replica():
    """compute_slice over a B200 replica that is still filling: the RSDP
    server reads its verified item prefix from the device watermarks -- a
    query answers progress 0 while nothing landed, a pull returns no bytes,
    and once the fill ran both see every item (transport.cpp:32-49,
    transport_stream.cpp:355-411)."""
    import socket
    import struct
    dev = torch.device("cuda:0")
    with Cluster() as cl:
        port = cl.listen()
        tb = _bufs(dev, seed=31)
        t = _open(cl, "T", tb)
        assert t.publish(1).status == Status.ok
        a = cl.open("m", "A", 1, tiny_threshold=1 << 20, grid_sms=32)
        ab = _bufs(dev)
        for i, b in enumerate(ab):
            assert a.register_tensor(0, f"w{i}", b) == Status.ok
        assert a.connect() == Status.ok
        assert a.server_replicate("latest").status == Status.ok
        assert a.transfer_bind(1) == Status.ok  # serving its empty fill

        c = socket.create_connection(("127.0.0.1", port))

        def recv_n(n):
            out = b""
            while len(out) < n:
                k = c.recv(n - len(out))
                assert k
                out += k
            return out

        def body(min_or_off, maxb=None):
            b = (b"\x01\x02" + struct.pack(">I", 1) + b"m" + b"\x02\x02" + struct.pack(">I", 1) + b"A" +
                 b"\x03\x01" + struct.pack(">Q", 1) + b"\x04\x01" + struct.pack(">Q", 0) +
                 b"\x05\x01" + struct.pack(">Q", min_or_off))
            return b + (b"\x06\x01" + struct.pack(">Q", maxb) if maxb is not None else b"")

        def query(min_items):
            q = body(min_items)
            c.sendall(struct.pack(">IHHQ", 0x52534450, 1, 3, len(q)) + q)
            assert struct.unpack(">IHHQ", recv_n(16))[2] == 4
            return struct.unpack(">BQB", recv_n(10))

        def pull(off, maxb):
            q = body(off, maxb)
            c.sendall(struct.pack(">IHHQ", 0x52534450, 1, 1, len(q)) + q)
            _, _, kind, blen = struct.unpack(">IHHQ", recv_n(16))
            st, prog, comp, plen = struct.unpack(">BQBQ", recv_n(18))
            return st, prog, comp, recv_n(plen)

        assert query(1) == (0, 0, 0)  # long-polled ~1 s: nothing verified yet
        st, prog, comp, payload = pull(0, 1 << 20)
        assert (st, prog, comp, len(payload)) == (0, 0, 0, 0)
        assert a.transfer_launch() == Status.ok
        assert a.transfer_wait() == [(Status.ok, 0)]
        st, prog, comp = query(10 ** 6)
        assert st == 0 and prog == 3  # w0, the group holding w1, w2 -- all verified
        total = sum(x.numel() for x in ab)
        got = b""
        while len(got) < total:
            st, prog, comp, payload = pull(len(got), total - len(got))
            assert st == 0 and payload
            got += payload
        # the item stream: big items in registration order, the group (w1) at
        # its first member's position -- here w0, group(w1), w2
        want = b"".join(x.cpu().numpy().tobytes() for x in tb)
        assert got == want
        a.transfer_finish(1, True)
        c.close()


def test_cross_datacenter_seed_over_tcp():
    """The realistic seeding case: the other datacenter's source is reached
    over the wire.  The seed fill receives its frames into pinned host
    memory and the pull kernel verifies them into the seed lane (host to
    host through the SM path); the owner then consumes the seed locally."""
    dev = torch.device("cuda:0")
    with Cluster() as cl:
        port = cl.listen()
        ep = f"tcp:127.0.0.1:{port}"
        tb = _bufs(dev, seed=31)
        t = _open(cl, "trainer", tb, ep, datacenter="dc1")
        assert t.publish(1).status == Status.ok
        fb = _bufs(dev)
        f = _open(cl, "far", fb, ep, datacenter="dc2", offload_seed=True)
        res = f.update()
        assert res.status == Status.ok and not res.changed, res
        assert f.seed_lanes() == [1]
        assert cl.view("m", "far+seed@1")["lifecycle"] == "published"
        res = f.update()
        assert res.status == Status.ok and res.changed and res.version == 1, res
        torch.cuda.synchronize()
        for a, b in zip(tb, fb):
            assert torch.equal(a, b)
        assert np.array_equal(f.chunk_digests(0), t.chunk_digests(0))
        st = f.stats()
        total = sum(b.numel() for b in tb)
        assert st.bytes_pulled_cross_dc == total and st.bytes_copied_local == total


def test_member_cut_groups_stream_over_tcp():
    """A replica whose packed groups are cut member by member (regions with
    slice geometry; layout.hpp member rule) streams over the B200 TCP plane:
    the header carries each member-cut item's runs, frames are cut at its
    batch boundaries, and the reader lands the bytes and the chunk table."""
    dev = torch.device("cuda:0")
    with Cluster() as cl:
        port = cl.listen()
        ep = f"tcp:127.0.0.1:{port}"
        sizes = [(1 << 20) + 4096 * 7, 6000, 4096, 333, 70000]
        t = cl.open("m", "trainer", 1, tiny_threshold=64 << 10)
        r = cl.open("m", "reader", 1, tiny_threshold=64 << 10)
        tb, rb = [], []
        from paper_2604_09107_b200 import ros
        for i, n in enumerate(sizes):
            a = torch.zeros(n, dtype=torch.uint8, device=dev)
            ros.synth_bf16(a[: n // 2 * 2], 40 + i)
            b = torch.zeros(n, dtype=torch.uint8, device=dev)
            tb.append(a)
            rb.append(b)
            g = (1, n, 0, 1, 0, n)  # a [1 x n] tensor held whole
            assert t.register_slice(0, f"w{i}", a, g) == Status.ok
            assert r.register_slice(0, f"w{i}", b, g) == Status.ok
        t.set_endpoint(0, ep)
        assert t.publish(1).status == Status.ok
        res = r.replicate(wait_s=20.0)
        assert res.status == Status.ok, res
        torch.cuda.synchronize()
        for a, b in zip(tb, rb):
            assert torch.equal(a, b)
        assert np.array_equal(r.chunk_digests(0), t.chunk_digests(0))
