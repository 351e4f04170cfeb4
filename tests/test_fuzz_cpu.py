"""CPU: hostile and malformed inputs at the library's parsers.

* Manifest bytes (TensorManifest::decode, manifest.cpp:103-173): the
  registry accepts a mutated manifest exactly when the reference decoder
  accepts it (oracle/_ref), and never crashes.
* The TCP data plane (stream.cpp, rsdp.cpp): random frames -- the B200
  stream handshake, the reference RSDP header with garbage bodies, plain
  noise -- never take the server down; it keeps answering a well-formed
  RSDP query afterwards.
"""
import ctypes as C
import socket
import struct

import pytest
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

from paper_2604_09107_b200._lib import lib
from paper_2604_09107_b200.ros import Cluster, Status


def _valid_manifest(oracle):
    names = ["a.weight", "b.weight", "c.bias", "d.norm"]
    lens = [3 << 20, 5000, 256, 4096]
    ng, g, off = oracle.assemble(lens)
    return oracle.manifest_encode(names, lens, [0x11, 0x22, 0x33, 0x44], g, off, ng, [0x55] * ng)


def _ref_decodes(ref, data: bytes) -> bool:
    lib_ref = ref.ref()
    lib_ref.ref_manifest_items.restype = C.c_long
    return lib_ref.ref_manifest_items(data, len(data), None, 0) >= 0


@pytest.fixture(scope="module")
def reg():
    cl = Cluster()
    yield cl
    cl.close()


_counter = [0]


def _publish(cl, data: bytes) -> int:
    _counter[0] += 1
    model = f"m{_counter[0]}".encode()  # a fresh model: no version 1 defined yet
    eps = (C.c_char_p * 1)(b"ep:x")
    assert lib.rs_server_open(cl.h, model, b"r", 1, b"dc0", C.cast(eps, C.c_void_p), b"", None, None,
                              None, None) == 0
    arr = (C.c_char_p * 1)(data)
    lens = (C.c_size_t * 1)(len(data))
    return lib.rs_server_publish(cl.h, model, b"r", 1, 1, C.cast(arr, C.c_void_p), C.cast(lens, C.c_void_p),
                                 None, None)


mutation = st.lists(st.tuples(st.integers(0, 10_000), st.integers(0, 255)), min_size=1, max_size=4)


@settings(max_examples=300, deadline=None, suppress_health_check=[HealthCheck.function_scoped_fixture])
@given(muts=mutation, cut=st.one_of(st.none(), st.integers(0, 10_000)),
       tail=st.binary(max_size=8))
def test_manifest_decoder_accepts_what_the_reference_accepts(ref, reg, muts, cut, tail):
    base = bytearray(_valid_manifest(ref))
    for pos, val in muts:
        base[pos % len(base)] = val
    data = bytes(base[: cut % (len(base) + 1)] if cut is not None else base) + tail
    rc = _publish(reg, data)
    assert rc in (Status.ok, Status.manifest_conflict), rc
    assert (rc == Status.ok) == _ref_decodes(ref, data), data.hex()


def test_valid_manifest_publishes(ref, reg):
    assert _publish(reg, _valid_manifest(ref)) == Status.ok


# ---- TCP data plane ----------------------------------------------------------

def _rsdp_query(port, replica=b"nope"):
    body = (b"\x01\x02" + struct.pack(">I", 1) + b"m" + b"\x02\x02" + struct.pack(">I", len(replica)) +
            replica + b"\x03\x01" + struct.pack(">Q", 1) + b"\x04\x01" + struct.pack(">Q", 0) +
            b"\x05\x01" + struct.pack(">Q", 1))
    c = socket.create_connection(("127.0.0.1", port), timeout=10)
    c.sendall(struct.pack(">IHHQ", 0x52534450, 1, 3, len(body)) + body)
    hdr = b""
    while len(hdr) < 16:
        k = c.recv(16 - len(hdr))
        assert k, "server closed the connection"
        hdr += k
    c.close()
    return struct.unpack(">IHHQ", hdr)


def _blast(port, payload: bytes):
    try:
        c = socket.create_connection(("127.0.0.1", port), timeout=2)
        c.settimeout(0.3)
        c.sendall(payload)
        try:
            c.recv(64)
        except OSError:
            pass
        c.close()
    except OSError:
        pass


@pytest.fixture(scope="module")
def server():
    cl = Cluster()
    port = cl.listen()
    yield port
    cl.close()


@settings(max_examples=150, deadline=None, suppress_health_check=[HealthCheck.function_scoped_fixture])
@given(kind=st.sampled_from(["noise", "rsdp", "stream"]), blob=st.binary(max_size=512),
       ver=st.integers(0, 3), mtype=st.integers(0, 9), blen=st.integers(0, 1 << 40))
def test_tcp_server_survives_malformed_frames(server, kind, blob, ver, mtype, blen):
    if kind == "rsdp":
        payload = struct.pack(">IHHQ", 0x52534450, ver, mtype, blen) + blob
    elif kind == "stream":
        payload = struct.pack("<II", 0x52534231, len(blob) * 7) + blob
    else:
        payload = blob
    _blast(server, payload)


def test_tcp_server_answers_after_the_fuzz(server):
    magic, ver, kind, blen = _rsdp_query(server)
    assert (magic, ver, kind) == (0x52534450, 1, 4)  # a query response


# ---- the operation log server (oplog.cpp) ------------------------------------

@pytest.fixture(scope="module")
def logsrv():
    from paper_2604_09107_b200.shared import LogServer
    log = LogServer()
    yield log
    log.close()


@settings(max_examples=100, deadline=None, suppress_health_check=[HealthCheck.function_scoped_fixture])
@given(blob=st.binary(max_size=256), kind=st.integers(0, 5), n=st.integers(0, 1 << 40))
def test_oplog_server_survives_malformed_requests(logsrv, blob, kind, n):
    payload = struct.pack("<II", 0x474C5352, kind) + struct.pack("<Q", n) + blob
    _blast(logsrv.port, payload if kind % 2 else blob)


def test_oplog_sequences_appends_after_the_fuzz(logsrv):
    from paper_2604_09107_b200.shared import SharedCluster
    sc = SharedCluster("127.0.0.1", logsrv.port)
    try:
        sc.sync()
        assert sc.applied >= 1
    finally:
        sc.close()
