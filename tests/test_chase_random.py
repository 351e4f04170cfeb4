"""GPU: randomized chains of readers chasing each other (SURVEY.md §8a
compute_slice / pipeline copies).  Seeded random tensor sets (a few bytes to
tens of MiB, random tiny thresholds and chunk sizes); three readers
replicate at once, so the planner chains them and each fill chases the
watermarks of the copy ahead of it while that copy is still landing.  On a
one-GPU box their persistent grids are capped (48 SMs each) so the kernels
co-reside.  Every reader must land the trainer's bytes and the trainer's
chunk-digest table."""
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _case(seed):
    rng = np.random.default_rng(20_000 + seed)
    tiny = int([64 << 10, 1 << 20, 2 << 20][int(rng.integers(0, 3))])
    chunk = int([2048, 4096, 16384][int(rng.integers(0, 3))])
    sizes = [int(rng.integers(1, 64 << 20)) if rng.random() < 0.4 else int(rng.integers(1, tiny))
             for _ in range(int(rng.integers(2, 12)))]
    return sizes, tiny, chunk


@pytest.mark.parametrize("seed", range(10))
def test_random_chained_readers_chase(seed):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2604_09107_b200 import ros
    from paper_2604_09107_b200.ros import Cluster, Status
    sizes, tiny, chunk = _case(seed)
    ngpu = torch.cuda.device_count()
    names = ["trainer", "r1", "r2", "r3"]
    with Cluster() as cl:
        hs, bufs = {}, {}
        for i, r in enumerate(names):
            dev = torch.device("cuda", i % ngpu)
            cfg = dict(tiny_threshold=tiny, chunk_bytes=chunk)
            if i and ngpu == 1:
                cfg["grid_sms"] = 48
            hs[r] = cl.open("m", r, 1, **cfg)
            bufs[r] = []
            for k, n in enumerate(sizes):
                t = torch.zeros(n, dtype=torch.uint8, device=dev)
                if i == 0:
                    ros.synth_bf16(t[: n // 2 * 2], 500 * seed + k)
                    if n % 2:
                        t[-1] = k
                bufs[r].append(t)
                assert hs[r].register_tensor(0, f"w{k}", t) == Status.ok
        torch.cuda.synchronize()
        assert hs["trainer"].publish(1).status == Status.ok
        results = {}

        def run(r):
            results[r] = hs[r].replicate(wait_s=60.0)

        ths = [threading.Thread(target=run, args=(r,)) for r in names[1:]]
        for th in ths:
            th.start()
        for th in ths:
            th.join()
        assert all(v.status == Status.ok for v in results.values()), (seed, results)
        srcs = [a.src for a in cl.assigns()]
        assert len(set(srcs)) == len(srcs) and "trainer" in srcs, srcs  # a chain
        table = hs["trainer"].chunk_digests(0)
        for r in names[1:]:
            for a, b in zip(bufs["trainer"], bufs[r]):
                assert torch.equal(a.cpu(), b.cpu()), (seed, r)
            assert np.array_equal(hs[r].chunk_digests(0), table), (seed, r)
