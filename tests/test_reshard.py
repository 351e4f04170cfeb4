"""TP/FSDP reshard on pull (K4, NEW: no reference counterpart).

CPU: the product's chunk rule equals the oracle restatement; the planner
gives resharding readers complete sources of another slicing and lets
same-slicing readers chase them.  GPU: TP-1 -> TP-2, FSDP-4 -> TP-2 and a
TP-2 reader chasing another TP-2 reader land exactly the numpy slices of
the trainer's tensors, with chunk digests equal to the oracle's."""
import ctypes as C

import numpy as np
import pytest

from paper_2604_09107_b200._lib import lib
from paper_2604_09107_b200.ros import Cluster, Status, tp_slice

# mini Llama: (name, shape, TP split dim)
HID, KV, FFN, VOCAB = 512, 128, 1408, 1000


def mini_llama(layers=2):
    t = [("model.embed_tokens.weight", (VOCAB, HID), 0)]
    for i in range(layers):
        p = f"model.layers.{i}."
        t += [(p + "self_attn.q_proj.weight", (HID, HID), 0),
              (p + "self_attn.k_proj.weight", (KV, HID), 0),
              (p + "self_attn.v_proj.weight", (KV, HID), 0),
              (p + "self_attn.o_proj.weight", (HID, HID), 1),
              (p + "mlp.gate_proj.weight", (FFN, HID), 0),
              (p + "mlp.up_proj.weight", (FFN, HID), 0),
              (p + "mlp.down_proj.weight", (HID, FFN), 1),
              (p + "input_layernorm.weight", (HID,), None),
              (p + "post_attention_layernorm.weight", (HID,), None)]
    t += [("model.norm.weight", (HID,), None), ("lm_head.weight", (VOCAB, HID), 0)]
    return t


def numel(shape):
    n = 1
    for d in shape:
        n *= d
    return n


# ------------------------------------------------------------------- CPU
def test_chunk_rule_matches_oracle(oracle):
    shapes = [(8192, 4096), (4096, 14336), (128256, 4096), (5120, 27648), (1024, 4096), (512, 1408),
              (5120,), (1000, 512), (3, 7), (33, 100)]
    for shape in shapes:
        for tp in (1, 2, 4, 8):
            for dim in (0, 1, None):
                if len(shape) == 1 and dim == 1:
                    continue
                g = tp_slice(shape, 2, dim, tp, 0)
                for align in (1, 2, 4, 8):
                    for cb in (512, 4096, 65536):
                        assert lib.rs_chunk_len_for(g[1], g[5], cb, align) == \
                            oracle.chunk_len_for(g[1], g[5], cb, align), (shape, tp, dim, align, cb)


def test_tp_slice_covers_tensor():
    for shape in [(1000, 512), (512,), (512, 1408)]:
        for dim in (0, 1, None):
            if len(shape) == 1 and dim == 1:
                continue
            parts = [tp_slice(shape, 2, dim, 2, r) for r in range(2)]
            assert sum(p[3] * p[5] for p in parts) == (numel(shape) * 2 * (1 if dim is not None else 2))


def _open(cl, replica, shards, key, dman=None, dlay=None):
    eps = (C.c_char_p * shards)(*[f"ep:{replica}:{i}".encode() for i in range(shards)])
    if dman:
        pm = (C.c_char_p * shards)(*dman)
        pl = (C.c_size_t * shards)(*[len(x) for x in dman])
        qm = (C.c_char_p * shards)(*dlay)
        ql = (C.c_size_t * shards)(*[len(x) for x in dlay])
        args = (C.cast(pm, C.c_void_p), C.cast(pl, C.c_void_p), C.cast(qm, C.c_void_p),
                C.cast(ql, C.c_void_p))
    else:
        args = (None, None, None, None)
    assert lib.rs_server_open(cl.h, b"m", replica.encode(), shards, b"dc0", C.cast(eps, C.c_void_p),
                              key.encode(), *args) == 0


def test_planner_reshard_and_same_slicing_chain(oracle):
    cl = Cluster()
    ng, g, off = oracle.assemble([1 << 20])
    man = oracle.manifest_encode(["w"], [1 << 20], [5], g, off, ng, [])
    half = oracle.manifest_encode(["w"], [1 << 19], [0], g, off, ng, [])
    _open(cl, "trainer", 1, "")
    arr = (C.c_char_p * 1)(man)
    lens = (C.c_size_t * 1)(len(man))
    assert lib.rs_server_publish(cl.h, b"m", b"trainer", 1, 1, C.cast(arr, C.c_void_p),
                                 C.cast(lens, C.c_void_p), None, None) == 0
    _open(cl, "tp2a", 2, "Lhalf", [half, half], [b"", b""])
    _open(cl, "tp2b", 2, "Lhalf", [half, half], [b"", b""])
    _open(cl, "plain", 1, "")
    for r in ("tp2a", "tp2b", "plain"):
        assert lib.rs_server_replicate(cl.h, b"m", r.encode(), b"latest") == 0
    got = [(a.replica, a.src) for a in cl.assigns()]
    # tp2a reshards from the trainer; tp2b (same slicing) chases tp2a's fill;
    # the plain reader is served item-for-item by the trainer
    assert got == [("tp2a", "trainer"), ("tp2b", "tp2a"), ("plain", "trainer")]
    # a plain reader never reshards: with only a differently sliced copy left
    # it gets no source
    _open(cl, "plain2", 1, "")
    cl.close()


# ------------------------------------------------------------------- GPU
torch = pytest.importorskip("torch")


def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _trainer_tensors(dev, tensors, seed0=100):
    from paper_2604_09107_b200 import ros
    full = {}
    for i, (n, shape, _) in enumerate(tensors):
        t = torch.empty(numel(shape) * 2, dtype=torch.uint8, device=dev)
        ros.synth_bf16(t, seed0 + i)
        full[n] = t
    return full


def _reader_items(oracle, tensors, shard_geos, full_host, tiny, chunk=4096, align=2):
    """Oracle view of one reader shard: manifest items (bytes) and chunk lens."""
    names = [n for n, _, _ in tensors]
    data = [oracle.slice_bytes(full_host[n], shard_geos[n]) for n in names]
    lens = [d.nbytes for d in data]
    ng, g, off = oracle.assemble(lens, tiny, 64 << 20)
    items, clens, seen = [], [], set()
    for e in range(len(names)):
        if g[e] < 0:
            items.append(data[e])
            geo = shard_geos[names[e]]
            clens.append(oracle.chunk_len_for(geo[1], geo[5], chunk, align))
        elif g[e] not in seen:
            # a packed group of regions with geometry is cut member by member
            # (layout.hpp member rule): each member is its own run of chunks
            seen.add(g[e])
            members = sorted((int(off[k]), k) for k in range(len(names)) if g[k] == g[e])
            for _, k in members:
                geo = shard_geos[names[k]]
                items.append(data[k])
                clens.append(oracle.chunk_len_for(geo[1], geo[5], chunk, align))
    enc = bytearray(oracle.manifest_encode(names, lens, [0] * len(names), g, off, ng, [0] * ng))
    enc[19] = 2  # derived-layout digest algorithm tag (field 2)
    return data, items, clens, bytes(enc)


def _publish_sharded(cl, name, dev, tensors, full, shards, split_of, tiny):
    h = cl.open("m", name, shards, tiny_threshold=tiny)
    keep = []
    for s in range(shards):
        for n, shape, dim in tensors:
            geo = split_of(shape, dim, s)
            rows, w, r0, nr, c0, nc = geo
            src = full[n].view(rows, w)[r0:r0 + nr, c0:c0 + nc].contiguous().view(-1)
            keep.append(src)
            assert h.register_slice(s, n, src, geo) == Status.ok
    return h, keep


def _reader_tp2(cl, name, dev, tensors, tiny):
    h = cl.open("m", name, 2, tiny_threshold=tiny)
    bufs, geos = {}, [{}, {}]
    for s in range(2):
        for n, shape, dim in tensors:
            geo = tp_slice(shape, 2, dim, 2, s)
            geos[s][n] = geo
            t = torch.zeros(geo[3] * geo[5], dtype=torch.uint8, device=dev)
            bufs[(s, n)] = t
            assert h.register_slice(s, n, t, geo) == Status.ok
    return h, bufs, geos


def _check_reader(oracle, h, bufs, geos, tensors, full, tiny):
    full_host = {n: t.cpu().numpy() for n, t in full.items()}
    for s in range(2):
        data, items, clens, enc = _reader_items(oracle, tensors, geos[s], full_host, tiny)
        for (n, _, _), d in zip(tensors, data):
            assert np.array_equal(bufs[(s, n)].cpu().numpy(), d), (s, n)
        assert h.manifest(s) == enc
        assert np.array_equal(h.chunk_digests(s), oracle.chunk_digests_lens(items, clens)), s


@pytest.mark.gpu
def test_tp1_to_tp2(oracle):
    _need_gpu()
    dev = torch.device("cuda:0")
    tiny = 64 << 10
    tensors = mini_llama()
    full = _trainer_tensors(dev, tensors)
    with Cluster() as cl:
        t, keep = _publish_sharded(cl, "trainer", dev, tensors, full, 1,
                                   lambda shape, dim, s: tp_slice(shape, 2, None, 1, 0), tiny)
        assert t.publish(1).status == Status.ok
        r, bufs, geos = _reader_tp2(cl, "tp2", dev, tensors, tiny)
        res = r.replicate()
        assert res.status == Status.ok, res
        assert [(a.replica, a.src) for a in cl.assigns()] == [("tp2", "trainer")]
        _check_reader(oracle, r, bufs, geos, tensors, full, tiny)
        st = r.stats()
        assert st.checksum_failures == 0 and st.items_verified > 0


@pytest.mark.gpu
def test_fsdp4_to_tp2_and_tp2_chain(oracle):
    _need_gpu()
    dev = torch.device("cuda:0")
    tiny = 64 << 10
    tensors = mini_llama()
    full = _trainer_tensors(dev, tensors, seed0=300)
    with Cluster() as cl:
        # FSDP2 Shard(0): 2-D tensors by row blocks, 1-D tensors by column blocks
        t, keep = _publish_sharded(cl, "fsdp", dev, tensors, full, 4,
                                   lambda shape, dim, s: tp_slice(shape, 2, 0, 4, s), tiny)
        assert t.publish(1).status == Status.ok
        r, bufs, geos = _reader_tp2(cl, "tp2a", dev, tensors, tiny)
        assert r.replicate().status == Status.ok
        _check_reader(oracle, r, bufs, geos, tensors, full, tiny)
        # a second TP-2 replica pulls item-for-item from the first
        r2, bufs2, geos2 = _reader_tp2(cl, "tp2b", dev, tensors, tiny)
        assert r2.replicate().status == Status.ok
        assert [(a.replica, a.src) for a in cl.assigns()][-1] == ("tp2b", "tp2a")
        _check_reader(oracle, r2, bufs2, geos2, tensors, full, tiny)


@pytest.mark.gpu
def test_reshard_detects_corrupt_source(oracle):
    _need_gpu()
    dev = torch.device("cuda:0")
    tiny = 64 << 10
    tensors = mini_llama(1)
    full = _trainer_tensors(dev, tensors, seed0=500)
    with Cluster() as cl:
        t, keep = _publish_sharded(cl, "trainer", dev, tensors, full, 1,
                                   lambda shape, dim, s: tp_slice(shape, 2, None, 1, 0), tiny)
        assert t.publish(1).status == Status.ok
        keep[4][100] ^= 0x5A  # corrupt o_proj in place after publish
        r, bufs, geos = _reader_tp2(cl, "tp2", dev, tensors, tiny)
        res = r.replicate(wait_s=5)
        assert res.status == Status.checksum_mismatch
        assert r.stats().checksum_failures >= 2


@pytest.mark.gpu
def test_member_cut_version_parked_in_host_memory(oracle):
    """A TP/FSDP trainer's packed groups are cut member by member (layout.hpp
    member rule).  When its version is parked in pinned host memory (a
    retention offload) a same-slicing reader pulls it from there: the
    member-cut items take the SM path (copy-engine frames assume uniform
    chunks) and land bit-exact with the trainer's chunk table."""
    _need_gpu()
    dev = torch.device("cuda:0")
    tiny = 64 << 10
    tensors = mini_llama(1)
    full = _trainer_tensors(dev, tensors, seed0=900)
    split = lambda shape, dim, s: tp_slice(shape, 2, 0, 2, s)  # noqa: E731  FSDP-2 row blocks
    with Cluster() as cl:
        w = cl.open("m", "watcher", 1)
        wt = torch.zeros(4096, dtype=torch.uint8, device=dev)
        assert w.register_tensor(0, "w0", wt) == Status.ok
        w.set_retention([0])
        assert w.connect() == Status.ok
        t, keep = _publish_sharded(cl, "trainer", dev, tensors, full, 2, split, tiny)
        assert t.publish(1).status == Status.ok
        tables = [t.chunk_digests(s) for s in range(2)]
        assert t.unpublish().status == Status.ok  # parks v1 in host memory
        assert t.lanes() == [1]
        r = cl.open("m", "reader", 2, tiny_threshold=tiny)
        bufs = {}
        for s in range(2):
            for n, shape, dim in tensors:
                geo = split(shape, dim, s)
                b = torch.zeros(geo[3] * geo[5], dtype=torch.uint8, device=dev)
                bufs[(s, n)] = (b, geo)
                assert r.register_slice(s, n, b, geo) == Status.ok
        res = r.replicate("1")
        assert res.status == Status.ok, res
        assert [(a.replica, a.src) for a in cl.assigns()][-1] == ("reader", "trainer+offload@1")
        torch.cuda.synchronize()
        for (s, n), (b, geo) in bufs.items():
            assert np.array_equal(b.cpu().numpy(), oracle.slice_bytes(full[n].cpu().numpy(), geo)), (s, n)
        for s in range(2):
            assert np.array_equal(r.chunk_digests(s), tables[s]), s
