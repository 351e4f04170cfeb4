"""CPU: dynamic membership through the registry's operation log
(paper_2604_09107_b200/shared.py; csrc/oplog.cpp).

The reference's clients dial its one metadata server whenever they start
(StreamServerHost / StreamControl, transport_stream.cpp:582-797).  Here each
process holds a registry replica that follows one sequenced log; a process
that starts after others have published replays the log and joins with the
same state.  Scenario (the reference chain, test_server_core.cpp:317-340):

  this process   hosts the log, opens "trainer", publishes v1
  process 1      starts afterwards: opens r1, replicates -> planned onto the
                 trainer; holds its fill open (still replicating)
  process 2      starts later still: opens r2, replicates -> planned onto r1,
                 a pipeline copy that is still filling (the elastic join)
  then r1 and r2 complete.  Every member's replica holds the same plan, the
  same listing, and the joiners never took part in a collective.
"""
import multiprocessing as mp
import os

import pytest

from tests.conftest import ROOT


def _manifest():
    import sys
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O
    names, lens = ["w0", "w1"], [4 << 20, 8192]
    ng, g, off = O.assemble(lens)
    return O.manifest_encode(names, lens, [0x1234, 0x5678], g, off, ng, [7] * ng)


def _member(name, port, go_complete, q):
    """A reader process that starts late, joins, replicates, completes."""
    import sys
    sys.path.insert(0, ROOT)
    try:
        from paper_2604_09107_b200.shared import SharedCluster
        sc = SharedCluster("127.0.0.1", port)
        sc.sync()  # replayed everything appended before it started
        seen_at_join = sorted((v, sorted(r)) for v, r in sc.listing("m").items())
        assert sc.op(("open", "m", name, 1, "dc0", [f"ep:{name}:0"], "", [], [])) == 0
        assert sc.op(("replicate", "m", name, "latest")) == 0
        done, st, v, _ = sc.result("m", name)
        src = sc._source("m", name)
        q.put((name, "planned", {"done": done, "status": int(st), "v": v, "src": src,
                                 "seen_at_join": seen_at_join}))
        go_complete.wait(60)
        assert sc.op(("complete", "m", name, 0, 0)) == 0
        sc.sync()
        q.put((name, "final", {"assigns": [(a.replica, a.src) for a in sc.assigns()],
                               "listing": {v: sorted(r) for v, r in sc.listing("m").items()},
                               "view": sc.local.view("m", name)}))
        go_complete.wait(60)
        sc.close()
    except Exception as e:  # pragma: no cover - surfaced by the parent
        import traceback
        q.put((name, "error", repr(e) + traceback.format_exc()))


def test_late_members_join_through_the_op_log():
    from paper_2604_09107_b200.shared import LogServer, SharedCluster
    log = LogServer()
    sc = SharedCluster("127.0.0.1", log.port)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ev = {n: ctx.Event() for n in ("r1", "r2")}
    ps = []
    try:
        assert sc.op(("open", "m", "trainer", 1, "dc0", ["ep:trainer:0"], "", [], [])) == 0
        assert sc.op(("publish", "m", "trainer", 1, [_manifest()], [])) == 0
        # r1 starts only now, after the publish
        ps.append(ctx.Process(target=_member, args=("r1", log.port, ev["r1"], q)))
        ps[-1].start()
        name, what, r1 = q.get(timeout=120)
        assert what == "planned", r1
        assert r1["done"] and r1["status"] == 0 and r1["v"] == 1 and r1["src"] == "trainer", r1
        assert r1["seen_at_join"] == [(1, ["trainer"])]
        # r2 starts while r1 is still replicating: planned onto r1 (pipeline copy)
        ps.append(ctx.Process(target=_member, args=("r2", log.port, ev["r2"], q)))
        ps[-1].start()
        name, what, r2 = q.get(timeout=120)
        assert what == "planned", r2
        assert r2["status"] == 0 and r2["src"] == "r1", r2
        sc.sync()
        assert sc.local.view("m", "r1")["lifecycle"] == "replicating"
        ev["r1"].set()
        ev["r2"].set()
        finals = {}
        for _ in range(2):
            name, what, f = q.get(timeout=120)
            assert what == "final", f
            finals[name] = f
        sc.sync()
        mine = [(a.replica, a.src) for a in sc.assigns()]
        assert mine == [("r1", "trainer"), ("r2", "r1")]
        for name, f in finals.items():
            assert f["assigns"] == mine, name  # the same plan in every replica
            assert f["view"]["lifecycle"] == "published"
        listing = {v: sorted(r) for v, r in sc.listing("m").items()}
        assert listing == {1: ["r1", "r2", "trainer"]}
        assert log.size > 8
    finally:
        for e in ev.values():
            e.set()
        for p in ps:
            p.join(timeout=30)
        sc.close()
        log.close()


def test_log_replays_in_order_for_a_member_that_starts_last():
    """A member that connects after 200 entries replays all of them and its
    follower applies each exactly once, in sequence order."""
    from paper_2604_09107_b200.shared import LogServer, SharedCluster
    log = LogServer()
    a = SharedCluster("127.0.0.1", log.port)
    try:
        assert a.op(("open", "m", "trainer", 1, "dc0", ["ep:t:0"], "", [], [])) == 0
        for v in range(1, 101):
            assert a.op(("publish", "m", "trainer", v, [_manifest()], [])) == 0
            assert a.op(("unpublish", "m", "trainer")) == 0
        assert a.op(("publish", "m", "trainer", 101, [_manifest()], [])) == 0
        b = SharedCluster("127.0.0.1", log.port)
        try:
            b.sync()  # entry 203: b replayed 0..202 and applied its own no-op
            assert b.applied == log.size == 203
            assert a._wait(lambda: a.applied == 203, 10)
            assert b.listing("m") == a.listing("m") == {101: {"trainer"}}
            assert b.local.trace().splitlines()[-5:] == a.local.trace().splitlines()[-5:]
        finally:
            b.close()
    finally:
        a.close()
        log.close()


def _tp2_part(shard, port, q, go):
    """One process of a TP-2 trainer group: its shard's parts of open and publish."""
    import sys
    sys.path.insert(0, ROOT)
    try:
        from paper_2604_09107_b200.shared import SharedCluster
        sc = SharedCluster("127.0.0.1", port)
        go.wait(60)
        part = {shard: {"ep": f"ep:T:{shard}", "hash": (0, False, False), "dm": b"", "dl": b""}}
        rc_open = sc.group_op(("m", "T", "open", 0), 2, part, {"dc": "dc0", "retain": []}, 30)
        rc_pub = sc.group_op(("m", "T", "publish", 0), 2, {shard: (_manifest(), b"")},
                             {"v": 1, "prov": False}, 30)
        sc.sync()
        q.put((shard, {"open": rc_open, "publish": rc_pub,
                       "listing": {v: sorted(r) for v, r in sc.listing("m").items()}}))
        go.wait(60)
        sc.close()
    except Exception as e:  # pragma: no cover
        import traceback
        q.put((shard, {"error": repr(e) + traceback.format_exc()}))


def test_group_transaction_joins_shards_from_two_processes():
    """server_core.cpp:298-591: the per-shard requests of a replica whose
    shards live in two processes join into one transaction; the replica
    opens and publishes once both parts are in, and a reader is then planned
    with a per-shard endpoint from each process (test_server_core.cpp:342-364)."""
    from paper_2604_09107_b200.shared import LogServer, SharedCluster
    log = LogServer()
    sc = SharedCluster("127.0.0.1", log.port)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    go = ctx.Event()
    ps = [ctx.Process(target=_tp2_part, args=(s, log.port, q, go)) for s in range(2)]
    try:
        for p in ps:
            p.start()
        go.set()
        res = dict(q.get(timeout=120) for _ in range(2))
        for s in range(2):
            assert "error" not in res[s], res[s]
            assert res[s]["open"] == 0 and res[s]["publish"] == 0, res[s]
            assert res[s]["listing"] == {1: ["T"]}
        sc.sync()
        assert sc.op(("open", "m", "R", 2, "dc0", ["ep:R:0", "ep:R:1"], "", [], [])) == 0
        assert sc.op(("replicate", "m", "R", "latest")) == 0
        eps = [sc.local.locate("m", "R", "latest", s)["source_endpoint"] for s in range(2)]
        assert eps == ["ep:T:0", "ep:T:1"]
    finally:
        for p in ps:
            p.join(timeout=30)
        sc.close()
        log.close()


def test_straggler_aborts_the_group_transaction():
    """A part that never arrives: the waiting member's abort entry wins the
    log order and every replica answers group_aborted; a part arriving after
    the abort changes nothing, and the next transaction starts clean."""
    from paper_2604_09107_b200.shared import LogServer, SharedCluster
    log = LogServer()
    a = SharedCluster("127.0.0.1", log.port)
    b = SharedCluster("127.0.0.1", log.port)
    try:
        part = lambda s: {s: {"ep": f"ep:T:{s}", "hash": (0, False, False), "dm": b"", "dl": b""}}  # noqa: E731
        key = ("m", "T", "open", 0)
        assert a.group_op(key, 2, part(0), {"dc": "dc0", "retain": []}, timeout=0.5) == 9  # group_aborted
        assert b.group_op(key, 2, part(1), {"dc": "dc0", "retain": []}, timeout=5) == 9
        b.sync()
        assert b.local.view("m", "T") is None and a.local.view("m", "T") is None
        key2 = ("m", "T", "open", 1)
        import threading
        out = {}
        th = threading.Thread(target=lambda: out.setdefault(
            "a", a.group_op(key2, 2, part(0), {"dc": "dc0", "retain": []}, timeout=30)))
        th.start()
        out["b"] = b.group_op(key2, 2, part(1), {"dc": "dc0", "retain": []}, timeout=30)
        th.join()
        assert out == {"a": 0, "b": 0}
        a.sync()
        assert a.local.view("m", "T")["lifecycle"] == "registered"
    finally:
        a.close()
        b.close()
        log.close()
