"""Fused bf16 -> fp8 e4m3 cast on pull (K5, NEW: no reference counterpart;
SURVEY.md §8 config 5).

A reader registers e4m3 regions for the version's bf16 entries; the pull
kernel verifies every chunk's XXH64 on the bf16 bytes it staged and lands
the saturating RNE cast (oracle ro_bf16_to_e4m3) instead of the bytes.  Such
a replica is terminal: the planner never hands it out as a source and it
cannot publish.

CPU: planner behaviour of terminal ("!") layout keys.  GPU: identity,
same-slicing TP-2 and TP-1 -> TP-2 reshard pulls land exactly
oracle.bf16_to_e4m3 of the trainer's bytes, with the bf16 chunk digests;
the slot path (RSB_NO_MAPS) and the LDGSTS kernel (RSB_PULL_KERNEL=ldg)
are re-run in subprocesses."""
import ctypes as C
import os
import subprocess
import sys

import numpy as np
import pytest

from paper_2604_09107_b200._lib import lib
from paper_2604_09107_b200.ros import Cluster, Status, tp_slice
from tests.test_reshard import _open, mini_llama, numel


# ------------------------------------------------------------------- CPU
def test_planner_terminal_never_serves(oracle):
    cl = Cluster()
    ng, g, off = oracle.assemble([1 << 20])
    man = oracle.manifest_encode(["w"], [1 << 20], [5], g, off, ng, [])
    _open(cl, "trainer", 1, "")
    arr = (C.c_char_p * 1)(man)
    lens = (C.c_size_t * 1)(len(man))
    assert lib.rs_server_publish(cl.h, b"m", b"trainer", 1, 1, C.cast(arr, C.c_void_p),
                                 C.cast(lens, C.c_void_p), None, None) == 0
    # "!" = a cast copy of the reference slicing "": pulled item-for-item
    _open(cl, "a8", 1, "!")
    _open(cl, "b16", 1, "")
    for r in ("a8", "b16"):
        assert lib.rs_server_replicate(cl.h, b"m", r.encode(), b"latest") == 0
    got = [(a.replica, a.src) for a in cl.assigns()]
    # b16 chases the trainer, never the (alphabetically first) fp8 copy
    assert got == [("a8", "trainer"), ("b16", "trainer")]
    # a terminal replica cannot publish
    _open(cl, "c8", 1, "!")
    assert lib.rs_server_publish(cl.h, b"m", b"c8", 2, 1, C.cast(arr, C.c_void_p),
                                 C.cast(lens, C.c_void_p), None, None) == int(Status.invalid_state)
    cl.close()


def test_oracle_cast_edges(oracle):
    # bf16 bit patterns: 0, -0, 1.0, 448, 464 (rounds to 448), 1e9 (sat), -inf,
    # +inf, NaN, smallest e4m3 subnormal 2^-9, half of it (ties to even -> 0)
    x = np.array([0x0000, 0x8000, 0x3F80, 0x43E0, 0x43E8, 0x4E6E, 0xFF80, 0x7F80, 0x7FC0,
                  0x3B00, 0x3A80], np.uint16)
    want = np.array([0x00, 0x80, 0x38, 0x7E, 0x7E, 0x7E, 0xFE, 0x7E, 0x7F, 0x01, 0x00], np.uint8)
    assert np.array_equal(oracle.bf16_to_e4m3(x), want)


# ------------------------------------------------------------------- GPU
torch = pytest.importorskip("torch")


def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _tensors():
    # mini Llama + a ragged entry (6600 B: a 2504-byte tail chunk) and an
    # entry of arbitrary bf16 bit patterns (NaN, inf, saturating, subnormal)
    return mini_llama(1) + [("odd.weight", (33, 100), None), ("wild.weight", (256, 1024), 1)]


def _full(dev, tensors, seed0=300):
    from paper_2604_09107_b200 import ros
    full = {}
    for i, (n, shape, _) in enumerate(tensors):
        t = torch.empty(numel(shape) * 2, dtype=torch.uint8, device=dev)
        if n == "wild.weight":
            rng = np.random.default_rng(7)
            t.copy_(torch.from_numpy(rng.integers(0, 256, t.numel(), dtype=np.uint8)))
        else:
            ros.synth_bf16(t, seed0 + i)
        full[n] = t
    return full


def _cast_of(oracle, host_bytes):
    return oracle.bf16_to_e4m3(np.ascontiguousarray(host_bytes).view(np.uint16))


def _fp8_region(dev, nbytes, misalign):
    """An e4m3 landing region of nbytes/2 bytes, optionally at an odd address."""
    n = nbytes // 2
    if not misalign:
        return torch.zeros(n, dtype=torch.uint8, device=dev)
    base = torch.zeros(n + 16, dtype=torch.uint8, device=dev)
    return base[3:3 + n]


@pytest.mark.gpu
@pytest.mark.parametrize("tiny", [4096, 64 << 10])
def test_identity_cast(oracle, tiny):
    _need_gpu()
    dev = torch.device("cuda:0")
    tensors = _tensors()
    full = _full(dev, tensors)
    with Cluster() as cl:
        t = cl.open("m", "trainer", 1, tiny_threshold=tiny)
        for n, _, _ in tensors:
            assert t.register_tensor(0, n, full[n]) == Status.ok
        assert t.publish(1).status == Status.ok
        r = cl.open("m", "fp8", 1, tiny_threshold=tiny)
        outs = {}
        for i, (n, _, _) in enumerate(tensors):
            outs[n] = _fp8_region(dev, full[n].numel(), misalign=(i % 5 == 4))
            assert r.register_cast(0, n, outs[n], full[n].numel()) == Status.ok
        assert r.layout_key == "!"
        res = r.replicate()
        assert res.status == Status.ok, res
        torch.cuda.synchronize()
        for n, _, _ in tensors:
            want = _cast_of(oracle, full[n].cpu().numpy())
            assert np.array_equal(outs[n].cpu().numpy(), want), n
        # verified on the bf16 bytes: the same chunk digests as the source
        assert np.array_equal(r.chunk_digests(0), t.chunk_digests(0))
        assert r.publish(2).status != Status.ok
        # a later bf16 reader is served by the trainer, never by the fp8 copy
        p = cl.open("m", "aa_bf16", 1, tiny_threshold=tiny)
        pb = {}
        for n, _, _ in tensors:
            pb[n] = torch.zeros_like(full[n])
            assert p.register_tensor(0, n, pb[n]) == Status.ok
        assert p.replicate().status == Status.ok
        assert [(a.replica, a.src) for a in cl.assigns()] == [("fp8", "trainer"),
                                                               ("aa_bf16", "trainer")]
        for n, _, _ in tensors:
            assert torch.equal(pb[n], full[n]), n


def _sharded_trainer(cl, full, tensors, tp, tiny, dim_of=lambda d: d):
    h = cl.open("m", "trainer", tp, tiny_threshold=tiny)
    keep = []
    for s in range(tp):
        for n, shape, dim in tensors:
            geo = tp_slice(shape, 2, dim_of(dim), tp, s)
            rows, w, r0, nr, c0, nc = geo
            src = full[n].view(rows, w)[r0:r0 + nr, c0:c0 + nc].contiguous().view(-1)
            keep.append(src)
            assert h.register_slice(s, n, src, geo) == Status.ok
    return h, keep


def _fp8_reader(cl, dev, tensors, tp, tiny, name="fp8"):
    h = cl.open("m", name, tp, tiny_threshold=tiny)
    outs, geos = {}, {}
    for s in range(tp):
        for n, shape, dim in tensors:
            geo = tp_slice(shape, 2, dim, tp, s)
            nbytes = geo[3] * geo[5]
            outs[(s, n)] = _fp8_region(dev, nbytes, misalign=False)
            geos[(s, n)] = geo
            assert h.register_cast(s, n, outs[(s, n)], nbytes, geo) == Status.ok
    return h, outs, geos


def _check_fp8(oracle, full, tensors, tp, outs, geos):
    torch.cuda.synchronize()
    for s in range(tp):
        for n, _, _ in tensors:
            sl = oracle.slice_bytes(full[n].cpu().numpy(), geos[(s, n)])
            assert np.array_equal(outs[(s, n)].cpu().numpy(), _cast_of(oracle, sl)), (s, n)


@pytest.mark.gpu
def test_same_slicing_tp2_cast(oracle):
    """Config 5 in miniature: shard i -> shard i, same slicing, cast on land."""
    _need_gpu()
    dev = torch.device("cuda:0")
    tensors, tiny = _tensors(), 64 << 10
    full = _full(dev, tensors)
    with Cluster() as cl:
        t, keep = _sharded_trainer(cl, full, tensors, 2, tiny)
        assert t.publish(1).status == Status.ok
        r, outs, geos = _fp8_reader(cl, dev, tensors, 2, tiny)
        assert r.layout_key == "!" + t.layout_key
        assert r.replicate().status == Status.ok
        # same slicing: item-for-item (no reshard), digests equal the source's
        for s in range(2):
            assert np.array_equal(r.chunk_digests(s), t.chunk_digests(s))
        _check_fp8(oracle, full, tensors, 2, outs, geos)


@pytest.mark.gpu
def test_reshard_tp1_to_tp2_cast(oracle):
    _need_gpu()
    dev = torch.device("cuda:0")
    tensors, tiny = _tensors(), 64 << 10
    full = _full(dev, tensors)
    with Cluster() as cl:
        t, keep = _sharded_trainer(cl, full, tensors, 1, tiny, dim_of=lambda d: None)
        assert t.publish(1).status == Status.ok
        r, outs, geos = _fp8_reader(cl, dev, tensors, 2, tiny)
        assert r.replicate().status == Status.ok
        _check_fp8(oracle, full, tensors, 2, outs, geos)
        # a bf16 TP-2 reader afterwards reshards from the trainer, not from
        # the fp8 copy of its slicing
        from tests.test_reshard import _reader_tp2
        b, bufs, bgeos = _reader_tp2(cl, "bf16", dev, tensors, tiny)
        assert b.replicate().status == Status.ok
        assert [(a.replica, a.src) for a in cl.assigns()][-1] == ("bf16", "trainer")


@pytest.mark.gpu
@pytest.mark.parametrize("env", ["RSB_NO_MAPS", "RSB_PULL_KERNEL"])
def test_cast_other_paths(env):
    """The slot (no tensor map) path of the TMA kernel and the LDGSTS kernel
    land the same casts (env read once per process: a subprocess each)."""
    _need_gpu()
    e = dict(os.environ)
    e[env] = "1" if env == "RSB_NO_MAPS" else "ldg"
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sel = [f"{__file__}::test_identity_cast", f"{__file__}::test_reshard_tp1_to_tp2_cast"]
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p",
                        "no:cacheprovider", *sel], cwd=root, env=e, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
