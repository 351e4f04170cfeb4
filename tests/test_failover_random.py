"""GPU: randomized corruption + failover (TransferTask item_failed / report /
re-pick, client_core.cpp:336-415; on_failure_report, server_core.cpp:
1291-1382).  A clean trainer T and a complete copy A of a random tensor set;
one random byte of one of A's big tensors (served in place) -- often in a
last partial chunk -- is flipped after A completed.  A reader
planned onto A must detect it (in-kernel chunk verification, one quiet
re-pull), report it, be re-planned onto T and land T's bytes exactly."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _case(seed):
    rng = np.random.default_rng(30_000 + seed)
    tiny = int([64 << 10, 1 << 20][int(rng.integers(0, 2))])
    sizes = [int(rng.integers(1, 24 << 20)) if rng.random() < 0.5 else int(rng.integers(1, tiny))
             for _ in range(int(rng.integers(2, 10)))]
    sizes.append(int(rng.integers(tiny, 24 << 20)))  # at least one item served in place
    # a big tensor: served from the registered region itself (a packed group
    # is served from its staging, which a flipped region byte does not touch)
    big = [i for i, n in enumerate(sizes) if n >= tiny]
    victim = big[int(rng.integers(0, len(big)))]
    pos = int(rng.integers(0, sizes[victim]))
    if rng.random() < 0.3:
        pos = sizes[victim] - 1  # the last byte: often a partial last chunk
    return sizes, tiny, victim, pos


@pytest.mark.parametrize("seed", range(12))
def test_random_corrupt_copy_fails_over_to_a_clean_source(seed):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2604_09107_b200 import ros
    from paper_2604_09107_b200.ros import Cluster, Status
    sizes, tiny, victim, pos = _case(seed)
    dev = torch.device("cuda:0")
    with Cluster() as cl:
        hs, bufs = {}, {}
        for i, r in enumerate(("T", "A", "R")):
            hs[r] = cl.open("m", r, 1, tiny_threshold=tiny, pull_timeout_s=2.0)
            bufs[r] = []
            for k, n in enumerate(sizes):
                t = torch.zeros(n, dtype=torch.uint8, device=dev)
                if r == "T":
                    ros.synth_bf16(t[: n // 2 * 2], 700 * seed + k)
                    if n % 2:
                        t[-1] = 0xA5
                bufs[r].append(t)
                assert hs[r].register_tensor(0, f"w{k}", t) == Status.ok
        torch.cuda.synchronize()
        assert hs["T"].publish(1).status == Status.ok
        assert hs["A"].replicate().status == Status.ok
        bufs["A"][victim][pos] ^= 0x5A  # A's copy goes bad after it verified
        torch.cuda.synchronize()
        res = hs["R"].replicate(wait_s=60.0)
        assert res.status == Status.ok, (seed, res)
        plan = [(a.replica, a.src) for a in cl.assigns() if a.replica == "R"]
        assert plan[0] == ("R", "A"), plan
        for a, b in zip(bufs["T"], bufs["R"]):
            assert torch.equal(a.cpu(), b.cpu()), (seed, victim, pos)
        st = hs["R"].stats()
        assert st.checksum_failures >= 1 and st.failure_reports >= 1, (seed, st)
        assert "failure_report" in cl.trace() and "reason=checksum" in cl.trace()
        assert np.array_equal(hs["R"].chunk_digests(0), hs["T"].chunk_digests(0))
