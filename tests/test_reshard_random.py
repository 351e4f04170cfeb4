"""GPU: randomized reshard cases (K4, with the K5 cast on some readers).

Seeded random models -- odd row counts and widths, 1-D and 2-D tensors,
random TP split dimensions, random tiny-tensor thresholds (so some slices
live in packed groups and some do not) -- published by an FSDP-k trainer
(k in 1, 2, 4; row blocks) and pulled by a TP-t reader (t in 2, 4) whose
shards all sit on cuda:0.  Every landed slice must equal the oracle's
numpy slice of the trainer's bytes (or its e4m3 cast), and the reader's
chunk-digest tables must equal the oracle's over the reader's own items."""
import numpy as np
import pytest

from paper_2604_09107_b200.ros import Cluster, Status, tp_slice

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _case(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(3, 12))
    tensors = []
    for i in range(n):
        if rng.random() < 0.25:
            shape = (int(rng.integers(1, 64)) * 4,)
            dim = None if rng.random() < 0.5 else 0
        else:
            shape = (int(rng.integers(1, 160)) * 4, int(rng.integers(1, 400)) * 4)
            dim = [0, 1, None][int(rng.integers(0, 3))]
        tensors.append((f"t{i}", shape, dim))
    fsdp = [1, 2, 4][int(rng.integers(0, 3))]
    tp = [2, 4][int(rng.integers(0, 2))]
    tiny = [4 << 10, 64 << 10, 1 << 20][int(rng.integers(0, 3))]
    cast = bool(rng.random() < 0.4)
    return tensors, fsdp, tp, tiny, cast


def _numel(shape):
    out = 1
    for d in shape:
        out *= d
    return out


def _expected_items(oracle, tensors, geos, full_host, tiny, chunk=4096, align=2):
    names = [n for n, _, _ in tensors]
    data = [oracle.slice_bytes(full_host[n], geos[n]) for n in names]
    lens = [d.nbytes for d in data]
    ng, g, off = oracle.assemble(lens, tiny, 64 << 20)
    items, clens, seen = [], [], set()
    for e in range(len(names)):
        if g[e] < 0:
            items.append(data[e])
            geo = geos[names[e]]
            clens.append(oracle.chunk_len_for(geo[1], geo[5], chunk, align))
        elif g[e] not in seen:
            # a packed group of regions with geometry is cut member by member
            # (layout.hpp member rule): each member is its own run of chunks
            seen.add(g[e])
            members = sorted((int(off[k]), k) for k in range(len(names)) if g[k] == g[e])
            for _, k in members:
                geo = geos[names[k]]
                items.append(data[k])
                clens.append(oracle.chunk_len_for(geo[1], geo[5], chunk, align))
    return data, items, clens


@pytest.mark.parametrize("seed", range(40))
def test_random_reshard(oracle, seed):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2604_09107_b200 import ros
    dev = torch.device("cuda:0")
    tensors, fsdp, tp, tiny, cast = _case(seed)
    full = {}
    for i, (n, shape, _) in enumerate(tensors):
        t = torch.empty(_numel(shape) * 2, dtype=torch.uint8, device=dev)
        ros.synth_bf16(t, 1000 * seed + i)
        full[n] = t
    torch.cuda.synchronize()
    with Cluster() as cl:
        tr = cl.open("m", "trainer", fsdp, tiny_threshold=tiny)
        keep = []
        for s in range(fsdp):
            for n, shape, _ in tensors:
                geo = tp_slice(shape, 2, 0, fsdp, s)  # FSDP2 Shard(0)
                rows, w, r0, nr, c0, nc = geo
                src = full[n].view(rows, w)[r0:r0 + nr, c0:c0 + nc].contiguous().view(-1)
                keep.append(src)
                assert tr.register_slice(s, n, src, geo) == Status.ok
        assert tr.publish(1).status == Status.ok
        rd = cl.open("m", "reader", tp, tiny_threshold=tiny)
        bufs, geos = {}, [dict() for _ in range(tp)]
        for s in range(tp):
            for n, shape, dim in tensors:
                geo = tp_slice(shape, 2, dim, tp, s)
                geos[s][n] = geo
                nbytes = geo[3] * geo[5]
                if cast:
                    b = torch.zeros(nbytes // 2, dtype=torch.uint8, device=dev)
                    assert rd.register_cast(s, n, b, nbytes, geo) == Status.ok
                else:
                    b = torch.zeros(nbytes, dtype=torch.uint8, device=dev)
                    assert rd.register_slice(s, n, b, geo) == Status.ok
                bufs[(s, n)] = b
        res = rd.replicate()
        assert res.status == Status.ok, (seed, res)
        torch.cuda.synchronize()
        full_host = {n: t.cpu().numpy() for n, t in full.items()}
        for s in range(tp):
            data, items, clens = _expected_items(oracle, tensors, geos[s], full_host, tiny)
            for (n, _, _), d in zip(tensors, data):
                want = oracle.bf16_to_e4m3(d.view(np.uint16)) if cast else d
                assert np.array_equal(bufs[(s, n)].cpu().numpy(), want), (seed, s, n)
            if not cast:  # a cast reader's table digests the bf16 bytes it verified
                assert np.array_equal(rd.chunk_digests(s), oracle.chunk_digests_lens(items, clens)), (seed, s)
        assert rd.stats().checksum_failures == 0
