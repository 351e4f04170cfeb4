"""CPU, world_size 2 over gloo: the replicated registry (dist.DistCluster)
computes identical plans on every rank, equal to the reference planner's."""
import json
import os
import socket

import pytest

from tests.conftest import ROOT, golden


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    import torch.distributed as dist

    import oracle as O
    from paper_2604_09107_b200.dist import DistCluster
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        dc = DistCluster()
        plan = json.load(open(golden("plans.json")))["chain7"]
        names = [n for n, _ in plan["tensors"]]
        lens = [l for _, l in plan["tensors"]]
        ng, g, off = O.assemble(lens)
        man = O.manifest_encode(names, lens, list(range(len(lens))), g, off, ng, [3] * ng)
        reps = plan["replicas"]
        # each rank opens half of the replicas; every rank mirrors all of them
        for i in range(0, len(reps), world):
            mine = reps[i + rank] if i + rank < len(reps) else None
            rc = dc.server_ops(None if mine is None else
                               ("open", "m", mine, 1, "dc0", [f"rank{rank}:{mine}"]))
            assert all(x in (None, 0) for x in rc)
        rc = dc.server_ops(("publish", "m", "trainer", 1, [man]) if rank == 0 else None)
        assert rc[0] == 0
        # simultaneous readers, arriving in registration order across ranks
        readers = reps[1:]
        for i in range(0, len(readers), world):
            mine = readers[i + rank] if i + rank < len(readers) else None
            dc.server_ops(None if mine is None else ("replicate", "m", mine, "latest"))
        # completions, then a failure report, in rank order everywhere
        for i in range(0, len(readers), world):
            mine = readers[i + rank] if i + rank < len(readers) else None
            dc.server_ops(None if mine is None else ("complete", "m", mine, 0, 0))
        q.put((rank, [(a.replica, a.version, a.src, a.src_serving) for a in dc.assigns()],
               dc.listing("m"), dc.local.trace()))
        dc.close()
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - surfaced by the parent
        q.put((rank, "error", repr(e), ""))
        raise


def test_replicated_registry_two_ranks_same_plan():
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = {}
    for _ in range(2):
        r = q.get(timeout=120)
        res[r[0]] = r
    for p in ps:
        p.join(timeout=60)
    assert all(res[r][1] != "error" for r in res), res
    plan = json.load(open(golden("plans.json")))["chain7"]
    want = [(a["replica"], a["version"], a["src"], a["src_serving"]) for a in plan["assigns"]]
    assert res[0][1] == res[1][1] == want
    assert res[0][2] == res[1][2]
    assert set(res[0][2][1]) == set(plan["replicas"])
    assert res[0][3] == res[1][3]  # byte-identical registry traces on both ranks


def test_replicated_registry_eight_ranks_same_plan():
    """The driver's 8-GPU scaling run in miniature: eight gloo ranks, one
    replica each (trainer + 7 readers replicating at once), every rank ends
    with the reference's chain plan and byte-identical registry traces."""
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    world = 8
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = {}
    for _ in range(world):
        r = q.get(timeout=300)
        res[r[0]] = r
    for p in ps:
        p.join(timeout=60)
    assert all(res[r][1] != "error" for r in res), res
    plan = json.load(open(golden("plans.json")))["chain7"]
    want = [(a["replica"], a["version"], a["src"], a["src_serving"]) for a in plan["assigns"]]
    assert all(res[r][1] == want for r in range(world))
    assert len({res[r][3] for r in range(world)}) == 1


class _FakeHandle:
    """The parts of ros.Handle DistCluster.open reads, for a replica whose
    shards are split across ranks (no device registrations on CPU)."""

    def __init__(self, model, replica, n, hashes):
        self.model, self.replica, self.num_shards = model, replica, n
        self.hashes = hashes

    def local_shards(self):
        return sorted(self.hashes)

    def shard_hash(self, s):
        return self.hashes[s]

    def derived(self, s, what):
        return b""

    def set_endpoint(self, s, e):
        pass


def _split_worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    import torch.distributed as dist

    import oracle as O
    from paper_2604_09107_b200.dist import DistCluster
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        dc = DistCluster()
        # trainer: shard r on rank r; reader: shard (r+1)%2 on rank r
        dc.open(_FakeHandle("m", "trainer", 2, {rank: (100 + rank, False, False)}),
                endpoints={rank: f"gpu{rank}"})
        dc.open(_FakeHandle("m", "reader", 2, {(rank + 1) % 2: (200 + rank, False, False)}),
                endpoints={(rank + 1) % 2: f"gpu{rank}"})
        ng, g, off = O.assemble([1 << 20])
        man = O.manifest_encode(["w"], [1 << 20], [7], g, off, ng, [])
        dc.server_ops(("publish", "m", "trainer", 1, [man, man]) if rank == 0 else None)
        eps = [dc.local.locate("m", "reader", "latest", s)["source_endpoint"] for s in range(2)]
        # a replica with a shard nobody registered cannot open
        try:
            dc.open(_FakeHandle("m", "half", 2, {0: (1, False, False)}) if rank == 0 else None)
            incomplete = "opened"
        except RuntimeError:
            incomplete = "refused"
        q.put((rank, eps, incomplete, dc.local.trace()))
        dc.close()
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - surfaced by the parent
        q.put((rank, "error", repr(e), ""))
        raise


def test_replica_split_across_ranks_merges_shards():
    """A TP-2 replica whose shards live on different ranks is one registry
    record with both shards' endpoints; every rank plans the same."""
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_split_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = {}
    for _ in range(2):
        r = q.get(timeout=120)
        res[r[0]] = r
    for p in ps:
        p.join(timeout=60)
    assert all(res[r][1] != "error" for r in res), res
    for r in range(2):
        assert res[r][1] == ["gpu0", "gpu1"]  # shard i is served from the rank holding it
        assert res[r][2] == "refused"
    assert res[0][3] == res[1][3]


def test_combine_layout_key():
    from paper_2604_09107_b200.ros import combine_layout_key as ck
    assert ck([(1, False, False), (2, False, False)]) == ""
    assert ck([(1, False, True), (2, False, False)]) == "!"
    k = ck([(1, True, False), (2, False, False)])
    assert k.startswith("L") and len(k) == 17
    assert ck([(1, True, True), (2, False, False)]) == "!" + k
    assert ck([(2, True, False), (1, False, False)]) != k  # shard order matters
