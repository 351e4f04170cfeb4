"""GPU: randomized publish/pull cases against the reference.

Seeded random tensor sets -- sizes from 1 byte to several MiB (ragged, odd,
exactly at the tiny threshold), random tiny thresholds and group targets,
random digest chunk sizes -- published and replicated through the C ABI
on cuda:0.  The publisher's manifest must be the reference library's
build_publish_payload bytes (oracle/_ref, or the C restatement without it);
the reader's bytes must equal the trainer's and both chunk-digest tables the
oracle's."""
import numpy as np
import pytest

from paper_2604_09107_b200.ros import Cluster, Status

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _case(seed):
    rng = np.random.default_rng(10_000 + seed)
    tiny = int([1 << 10, 64 << 10, 512 << 10, 2 << 20][int(rng.integers(0, 4))])
    target = int([tiny * 2, 1 << 20, 64 << 20][int(rng.integers(0, 3))])
    chunk = int([1024, 4096, 8192, 65536][int(rng.integers(0, 4))])
    sizes = []
    for _ in range(int(rng.integers(1, 25))):
        kind = rng.random()
        if kind < 0.15:
            sizes.append(int(rng.integers(1, 33)))                  # a few bytes
        elif kind < 0.25:
            sizes.append(tiny + int(rng.integers(-1, 2)))           # at the threshold
        elif kind < 0.7:
            sizes.append(int(rng.integers(33, tiny + 1)))           # tiny: packed
        else:
            sizes.append(int(rng.integers(tiny, 6 << 20)))          # big: an item of its own
    return [max(1, s) for s in sizes], tiny, target, chunk


@pytest.mark.parametrize("seed", range(30))
def test_random_publish_pull_matches_reference(oracle, seed):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    sizes, tiny, target, chunk = _case(seed)
    rng = np.random.default_rng(seed)
    host = [rng.integers(0, 256, n, dtype=np.uint8) for n in sizes]
    names = [f"layer{i}.w" for i in range(len(sizes))]
    dev = torch.device("cuda:0")
    cfg = dict(tiny_threshold=tiny, group_target=target, chunk_bytes=chunk)
    with Cluster() as cl:
        t = cl.open("m", "trainer", 1, **cfg)
        r = cl.open("m", "reader", 1, **cfg)
        tb, rb = [], []
        for n, a in zip(names, host):
            x = torch.from_numpy(a).to(dev)
            y = torch.zeros_like(x)
            tb.append(x)
            rb.append(y)
            assert t.register_tensor(0, n, x) == Status.ok
            assert r.register_tensor(0, n, y) == Status.ok
        assert t.publish(1).status == Status.ok
        res = r.replicate()
        assert res.status == Status.ok, (seed, res)
        torch.cuda.synchronize()
        for x, y in zip(tb, rb):
            assert torch.equal(x, y), seed
        want = (oracle.ref_build_manifest(names, host, tiny, target) if oracle.ref_available()
                else oracle.publish_manifest(names, host, tiny, target))
        assert t.manifest(0) == want, seed
        assert r.manifest(0) == want, seed
        ng, g, off = oracle.assemble(sizes, tiny, target)
        items, seen = [], set()
        for e in range(len(sizes)):
            if g[e] < 0:
                items.append(host[e])
            elif g[e] not in seen:
                seen.add(g[e])
                members = sorted((int(off[k]), k) for k in range(len(sizes)) if g[k] == g[e])
                items.append(np.concatenate([host[k] for _, k in members]))
        table = oracle.chunk_digests(items, chunk)
        assert np.array_equal(t.chunk_digests(0), table), seed
        assert np.array_equal(r.chunk_digests(0), table), seed


def test_many_tiny_tensors_match_reference(oracle):
    """3,000 tiny tensors (1 B - 5 KB) and two big ones: many packed groups,
    thousands of pack/unpack spans and K6 spans in one publish and pull."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    rng = np.random.default_rng(77)
    sizes = [int(x) for x in rng.integers(1, 5000, 3000)] + [5 << 20, (3 << 20) + 7]
    rng.shuffle(sizes)
    host = [rng.integers(0, 256, n, dtype=np.uint8) for n in sizes]
    names = [f"p{i}" for i in range(len(sizes))]
    tiny, target = 64 << 10, 1 << 20
    dev = torch.device("cuda:0")
    with Cluster() as cl:
        t = cl.open("m", "trainer", 1, tiny_threshold=tiny, group_target=target)
        r = cl.open("m", "reader", 1, tiny_threshold=tiny, group_target=target)
        tb, rb = [], []
        for n, a in zip(names, host):
            x = torch.from_numpy(a).to(dev)
            y = torch.zeros_like(x)
            tb.append(x)
            rb.append(y)
            assert t.register_tensor(0, n, x) == Status.ok
            assert r.register_tensor(0, n, y) == Status.ok
        assert t.publish(1).status == Status.ok
        assert r.replicate().status == Status.ok
        torch.cuda.synchronize()
        assert all(torch.equal(x, y) for x, y in zip(tb, rb))
        want = (oracle.ref_build_manifest(names, host, tiny, target) if oracle.ref_available()
                else oracle.publish_manifest(names, host, tiny, target))
        assert t.manifest(0) == want and r.manifest(0) == want
        assert np.array_equal(r.chunk_digests(0), t.chunk_digests(0))


@pytest.mark.parametrize("seed", range(10))
def test_random_cast_pull_matches_oracle(oracle, seed):
    """Fused bf16 -> e4m3 landing (the three-stage V15 shape) over random
    bf16 tensor sets: odd element counts, tensors that straddle the tiny
    threshold (packed members land as e4m3 through the group path)."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    rng = np.random.default_rng(40_000 + seed)
    tiny = int([64 << 10, 1 << 20][int(rng.integers(0, 2))])
    elems = [int(rng.integers(1, 3 << 20)) if rng.random() < 0.5 else int(rng.integers(1, tiny // 2))
             for _ in range(int(rng.integers(2, 10)))]
    host = [oracle.synth_bf16(900 * seed + i, n) for i, n in enumerate(elems)]
    dev = torch.device("cuda:0")
    with Cluster() as cl:
        t = cl.open("m", "trainer", 1, tiny_threshold=tiny)
        r = cl.open("m", "fp8", 1, tiny_threshold=tiny)
        outs = []
        for i, a in enumerate(host):
            x = torch.from_numpy(a.view(np.int16).copy()).to(dev)
            y = torch.zeros(a.size, dtype=torch.uint8, device=dev)
            outs.append(y)
            assert t.register_tensor(0, f"w{i}", x) == Status.ok
            assert r.register_cast(0, f"w{i}", y, a.nbytes) == Status.ok
        assert t.publish(1).status == Status.ok
        res = r.replicate()
        assert res.status == Status.ok, (seed, res)
        torch.cuda.synchronize()
        for a, y in zip(host, outs):
            assert np.array_equal(y.cpu().numpy(), oracle.bf16_to_e4m3(a)), seed
        assert np.array_equal(r.chunk_digests(0), t.chunk_digests(0))
