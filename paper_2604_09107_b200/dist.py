"""Multi-process ROS: one process per GPU, registry replicated on every rank.

The reference runs one metadata server that every client talks to
(ServerCore, server_core.cpp; Channel/ControlPlane, transport.hpp:23-43).
Here every rank holds a replica of the registry (csrc/registry.cpp) and the
ranks apply one operation log in one order: each collective call
all-gathers the per-rank operations (None = nothing to do) over a gloo
group and applies them in rank order, so every replica of the planner sees
the same request sequence and computes the same plan -- for simultaneous
readers exactly the order the reference's SimExecutor would (Appendix A of
SURVEY.md).  The data path never uses a collective: serve states (landing
buffers, chunk-digest tables, watermark words) travel as CUDA IPC handles
and readers pull them with the SM-driven kernel, chasing upstream
watermarks in device memory.

All methods except create() are collective over the group: every rank calls
them in the same order, passing its local handle (or None when it has no
part in that operation).
"""
from __future__ import annotations

import ctypes as C
from typing import Optional

from ._lib import lib
from .ros import Cluster, Handle, OpResult, Status, _read_bytes, check, combine_layout_key


def _b(s: str) -> bytes:
    return s.encode()


def _blob_arrays(blobs):
    arr = (C.c_char_p * max(len(blobs), 1))(*blobs)
    lens = (C.c_size_t * max(len(blobs), 1))(*[len(x) for x in blobs])
    return C.cast(arr, C.c_void_p), C.cast(lens, C.c_void_p), arr, lens


def lib_manifest(h, shard: int) -> bytes:
    """The shard's manifest bytes as held right now (provisional during an
    early publish; Handle.manifest waits for the final ones)."""
    return _read_bytes(lib.rs_manifest_now, h.h, shard)


def apply_op(c, o) -> int:
    """Applies one registry operation (see DistCluster.server_ops) to the
    registry replica `c` (an rs_cluster handle); returns its status code."""
    kind = o[0]
    if kind == "open":
        _, m, r, n, dc, eps = o[:6]
        key = o[6] if len(o) > 6 else ""
        dman = o[7] if len(o) > 7 else []
        dlay = o[8] if len(o) > 8 else []
        arr = (C.c_char_p * n)(*[_b(e) for e in eps])
        if dman:
            pm, pl, _k1, _k2 = _blob_arrays(dman)
            qm, ql, _k3, _k4 = _blob_arrays(dlay)
        else:
            pm = pl = qm = ql = None
        return lib.rs_server_open(c, _b(m), _b(r), n, _b(dc), C.cast(arr, C.c_void_p), _b(key),
                                  pm, pl, qm, ql)
    if kind == "publish":
        _, m, r, v, mans = o[:5]
        lays = o[5] if len(o) > 5 else []
        provisional = bool(o[6]) if len(o) > 6 else False  # an early publish
        pm, pl, _k1, _k2 = _blob_arrays(mans)
        if lays:
            qm, ql, _k3, _k4 = _blob_arrays(lays)
        else:
            qm = ql = None
        fn = lib.rs_server_publish_provisional if provisional else lib.rs_server_publish
        return fn(c, _b(m), _b(r), v, len(mans), pm, pl, qm, ql)
    if kind == "finalize":
        _, m, r, v, mans = o
        pm, pl, _k1, _k2 = _blob_arrays(mans)
        return lib.rs_server_finalize(c, _b(m), _b(r), v, len(mans), pm, pl)
    if kind == "add_layout":
        _, m, v, key, mans, lays = o
        pm, pl, _k1, _k2 = _blob_arrays(mans)
        qm, ql, _k3, _k4 = _blob_arrays(lays)
        return lib.rs_server_add_layout(c, _b(m), v, _b(key), len(mans), pm, pl, qm, ql)
    if kind == "unpublish":
        return lib.rs_server_unpublish(c, _b(o[1]), _b(o[2]))
    if kind == "retain":
        _, m, r, lags = o
        arr = (C.c_uint64 * max(len(lags), 1))(*lags)
        return lib.rs_server_set_retention(c, _b(m), _b(r), C.cast(arr, C.c_void_p), len(lags))
    if kind == "offload_confirm":
        _, m, r, shard, v, ok, ep = o
        return lib.rs_server_offload_confirm(c, _b(m), _b(r), shard, v, int(ok), _b(ep))
    if kind == "replicate":
        return lib.rs_server_replicate(c, _b(o[1]), _b(o[2]), _b(o[3]))
    if kind == "update":
        _, m, r, sp, cur = o
        return lib.rs_server_update(c, _b(m), _b(r), _b(sp), int(cur is not None), cur or 0)
    if kind == "complete":
        return lib.rs_server_complete(c, _b(o[1]), _b(o[2]), o[3], o[4])
    if kind == "seed_on":  # ClientConfig.offload_seed (OpenReq.offload_seed)
        return lib.rs_server_set_offload_seed(c, _b(o[1]), _b(o[2]), 1)
    if kind == "seed_complete":  # CompleteMsg, TransferRole::seed
        _, m, r, shard, outcome, v = o
        return lib.rs_server_seed_complete(c, _b(m), _b(r), shard, outcome, v)
    if kind == "report":
        return lib.rs_server_failure_report(c, _b(o[1]), _b(o[2]), o[3], _b(o[4]), o[5])
    if kind == "close":
        return lib.rs_server_close(c, _b(o[1]), _b(o[2]))
    raise ValueError(kind)

class DistCluster:
    def __init__(self, group=None, pipeline: bool = True, smart_skipping: bool = True):
        import torch.distributed as dist
        self.dist = dist
        self.rank = dist.get_rank()
        self.world = dist.get_world_size()
        self.pg = group if group is not None else dist.new_group(backend="gloo")
        self.local = Cluster(pipeline=pipeline, smart_skipping=smart_skipping)
        self._txn = {}  # id(handle) -> replicate_start state awaiting replicate_finish

    # ---- plumbing ----------------------------------------------------------
    def gather(self, obj):
        out = [None] * self.world
        self.dist.all_gather_object(out, obj, group=self.pg)
        return out

    def close(self):
        self.local.close()

    def _import_all(self, blobs):
        for r, bl in enumerate(blobs):
            if r == self.rank or not bl:
                continue
            for b in bl:
                check(lib.rs_serve_import(self.local.h, b, len(b)), "rs_serve_import")

    def _source(self, model, replica) -> str:
        return _read_bytes(lib.rs_cluster_source, self.local.h, _b(model), _b(replica)).decode()

    def server_ops(self, op):
        """Collective: all-gather one registry operation per rank (or None)
        and apply them to the local registry replica in rank order.  Ops:
        ("open", model, replica, shards, dc, endpoints[, layout_key]),
        ("publish", model, replica, version, [manifests][, [layouts]]),
        ("add_layout", model, version, layout_key, [manifests], [layouts]),
        ("unpublish", model, replica), ("replicate", model, replica, spec),
        ("update", model, replica, spec, current|None),
        ("complete", model, replica, shard, status),
        ("report", model, replica, shard, failed_replica, reason).
        Returns the per-rank return codes."""
        out = []
        for o in self.gather(op):
            out.append(None if o is None else self._apply(o))
        return out

    def _apply(self, o) -> int:
        return apply_op(self.local.h, o)

    def set_topology(self, endpoints, cost) -> None:
        """Local, but every rank must call it with the same arguments (the
        registry replicas must plan alike): rank 0's matrix is broadcast."""
        endpoints, cost = self.gather((list(endpoints), [list(r) for r in cost]))[0]
        self.local.set_topology(endpoints, cost)

    def result(self, model, replica):
        d, s, v, ch = C.c_int(), C.c_int(), C.c_uint64(), C.c_int()
        lib.rs_server_result(self.local.h, _b(model), _b(replica), C.byref(d), C.byref(s),
                             C.byref(v), C.byref(ch))
        return bool(d.value), Status(s.value), v.value, bool(ch.value)

    # ---- ops ---------------------------------------------------------------
    # A replica may span several ranks (a TP/FSDP group: one process per
    # GPU, each holding some of the replica's shards).  Every rank holding
    # shards of a replica passes its handle; the parts are merged per
    # replica (rank order) into the one registry operation the reference's
    # server would receive from that replica's client.
    def create(self, model: str, replica: str, num_shards: int = 1, **cfg) -> Handle:
        """Local: a handle to register tensors on, before the collective open()."""
        return self.local.open(model, replica, num_shards, **cfg)

    @staticmethod
    def _merge(parts):
        """{(model, replica): [part, ...]} in rank order (None parts skipped)."""
        out = {}
        for p in parts:
            if p is not None:
                out.setdefault((p["model"], p["replica"]), []).append(p)
        return out

    def open(self, h: Optional[Handle], endpoints=None, datacenter: str = "dc0") -> None:
        """Collective: every rank mirrors every opened replica's record (its
        endpoints per shard and slicing key, gathered from the ranks holding
        its shards).  endpoints: one per local shard (list) or {shard: ep}."""
        mine = None
        if h is not None:
            loc = h.local_shards()
            if endpoints is None:
                eps = {s: f"rank{self.rank}:{s}" for s in loc}
            elif isinstance(endpoints, dict):
                eps = dict(endpoints)
            else:
                eps = dict(zip(loc, endpoints))
            for sh, e in eps.items():
                h.set_endpoint(sh, e)
            hashes = {sh: h.shard_hash(sh) for sh in loc}
            geo = any(x[1] for x in hashes.values())
            derived = {sh: (h.derived(sh, 0), h.derived(sh, 1)) for sh in loc} if geo else {}
            mine = {"model": h.model, "replica": h.replica, "n": h.num_shards, "dc": datacenter,
                    "eps": eps, "hashes": hashes, "derived": derived,
                    "retain": list(getattr(h, "retain", []))}
        for (m, r), parts in self._merge(self.gather(mine)).items():
            n = parts[0]["n"]
            eps, hashes, derived = {}, {}, {}
            for p in parts:
                eps.update(p["eps"])
                hashes.update(p["hashes"])
                derived.update(p["derived"])
            if sorted(hashes) != list(range(n)):
                raise RuntimeError(f"open {m}/{r}: shards {sorted(hashes)} registered, {n} expected")
            key = combine_layout_key([hashes[i] for i in range(n)])
            dman = [derived[i][0] for i in range(n)] if derived else []
            dlay = [derived[i][1] for i in range(n)] if derived else []
            rc = self._apply(("open", m, r, n, parts[0]["dc"], [eps[i] for i in range(n)], key,
                              dman, dlay))
            assert rc == 0, (m, r, rc)
            retain = sorted({x for p in parts for x in p.get("retain", [])})
            if retain:
                assert self._apply(("retain", m, r, retain)) == 0

    def publish(self, h: Optional[Handle], version: int) -> Optional[OpResult]:
        mine = None
        if h is not None:
            check(lib.rs_prepare_publish(h.h, version), "rs_prepare_publish")
            mine = {"model": h.model, "replica": h.replica, "n": h.num_shards,
                    "provisional": h.publish_pending,
                    "shards": {s: (lib_manifest(h, s), h.layout(s)) for s in h.local_shards()}}
        rcs = {}
        for (m, r), parts in self._merge(self.gather(mine)).items():
            n = parts[0]["n"]
            sh = {}
            for p in parts:
                sh.update(p["shards"])
            if sorted(sh) != list(range(n)):
                rcs[(m, r)] = int(Status.invalid_argument)
                continue
            rcs[(m, r)] = self._apply(("publish", m, r, version, [sh[i][0] for i in range(n)],
                                       [sh[i][1] for i in range(n)],
                                       any(p.get("provisional") for p in parts)))
        blobs = None
        if h is not None:
            st = rcs[(h.model, h.replica)]
            lib.rs_commit_publish(h.h, version, st)
            if st == 0:
                blobs = [h.serve_export(s) for s in h.local_shards()]
        self._import_all(self.gather(blobs))
        if h is None:
            return None
        st = Status(rcs[(h.model, h.replica)])
        return OpResult(st, version if st == Status.ok else None)

    def _offload_first(self, h: Optional[Handle]) -> None:
        """Collective: replicas whose unpublish/update waits for a retention
        offload park the version in host memory (their ranks' local shards),
        confirm every shard, and every rank imports the offload lanes."""
        mine = None
        if h is not None:
            v = C.c_uint64()
            if lib.rs_server_offload_pending(self.local.h, _b(h.model), _b(h.replica), C.byref(v)):
                ok = lib.rs_offload_lanes(h.h, v.value) == 0
                loc = h.local_shards()
                blobs = [_read_bytes(lib.rs_lane_export, h.h, s, v.value) for s in loc] if ok else []
                mine = {"model": h.model, "replica": h.replica, "v": v.value, "ok": ok,
                        "eps": {s: f"host:{h.replica}:{s}" for s in loc}, "blobs": blobs}
        parts = self.gather(mine)
        if not any(parts):
            return
        for p in parts:
            if p is None:
                continue
            for s, ep in p["eps"].items():
                self._apply(("offload_confirm", p["model"], p["replica"], s, p["v"], p["ok"], ep))
        self._import_all([p["blobs"] if p else None for p in parts])

    def finalize(self, h: Optional[Handle]) -> None:
        """Collective: an early publish's ranks wait for their big-entry
        digests and every registry replica commits the final manifests."""
        mine = None
        if h is not None:
            v = h.current_version
            check(lib.rs_publish_finalize(h.h, 60.0), "rs_publish_finalize")
            mine = {"model": h.model, "replica": h.replica, "n": h.num_shards, "v": v,
                    "shards": {s: h.manifest(s) for s in h.local_shards()}}
        for (m, r), parts in self._merge(self.gather(mine)).items():
            sh = {}
            for p in parts:
                sh.update(p["shards"])
            n = parts[0]["n"]
            if sorted(sh) == list(range(n)):
                self._apply(("finalize", m, r, parts[0]["v"], [sh[i] for i in range(n)]))

    def unpublish(self, h: Optional[Handle]) -> Optional[OpResult]:
        mine = {"model": h.model, "replica": h.replica} if h is not None else None
        rcs = {k: self._apply(("unpublish",) + k) for k in self._merge(self.gather(mine))}
        self._offload_first(h)
        if h is None:
            return None
        done, s, _, _ = self.result(h.model, h.replica)
        rc = rcs[(h.model, h.replica)]
        st = Status(rc) if rc else s
        return OpResult(st if done else Status.timeout)

    def replicate(self, h: Optional[Handle], spec: str = "latest", update: bool = False,
                  max_rounds: int = 8) -> Optional[OpResult]:
        """Collective replicate/update: plan on every rank, bind + serve,
        exchange serve states, then every reader shard fills (kernels chase
        each other's watermarks), with failure reports applied collectively.
        A replica spanning several ranks completes only when all its shards
        verified.  = replicate_start + replicate_finish."""
        self.replicate_start(h, spec, update)
        return self.replicate_finish(h, max_rounds)

    def replicate_start(self, h: Optional[Handle], spec: str = "latest",
                        update: bool = False) -> None:
        """Collective first half: plan, bind, exchange serve states and LAUNCH
        the local shards' pull kernels; returns while they run.  Another
        replicate_start (a late joiner) may follow before replicate_finish."""
        mine = None
        if h is not None:
            mine = {"model": h.model, "replica": h.replica, "update": update, "spec": spec,
                    "cur": h.current_version}
        for (m, r), parts in self._merge(self.gather(mine)).items():
            p = parts[0]
            self._apply(("update", m, r, p["spec"], p["cur"]) if p["update"] else
                        ("replicate", m, r, p["spec"]))
        self._offload_first(h)
        txn = {"active": False, "result": None, "version": None, "changed": False,
               "loc": h.local_shards() if h is not None else [], "launched": False}
        if h is not None:
            d, s, v, ch = self.result(h.model, h.replica)
            cur = h.current_version
            if not d:
                txn["result"] = OpResult(Status.timeout)  # parked: no version yet
            elif s != Status.ok:
                txn["result"] = OpResult(s)
            elif update and not ch:
                txn["result"] = OpResult(Status.ok, v or cur, False)
            else:
                txn["version"], txn["changed"] = v, ch or not update
                rc = lib.rs_transfer_bind(h.h, v)
                if rc != 0:
                    txn["result"] = OpResult(Status(rc))
                else:
                    txn["active"] = True
        blobs = [h.serve_export(s) for s in txn["loc"]] if txn["active"] else None
        # one all-gather: the serve states to import, and every part's bind
        # outcome (a replica whose bind failed on one rank fails on all of its ranks)
        got = self.gather((blobs, (h.model, h.replica, txn["active"], txn["result"] is not None)
                           if h is not None else None))
        self._import_all([g[0] for g in got])
        bind = [g[1] for g in got]
        broken = {(b[0], b[1]) for b in bind if b is not None and b[3] and not b[2]}
        if txn["active"] and (h.model, h.replica) in broken:
            lib.rs_transfer_finish(h.h, txn["version"], 0)
            txn["result"] = OpResult(Status.transfer_failed)
            txn["active"] = False
        if txn["active"]:
            check(lib.rs_transfer_launch(h.h), "rs_transfer_launch")
            txn["launched"] = True
        if h is not None:
            self._txn[id(h)] = txn

    def progress(self, h: Handle, shard: int) -> tuple[int, int]:
        """Local: (verified batches, batches) of a running fill of one shard."""
        done, n = C.c_uint32(), C.c_uint32()
        check(lib.rs_transfer_progress(h.h, shard, C.byref(done), C.byref(n)))
        return done.value, n.value

    def replicate_finish(self, h: Optional[Handle], max_rounds: int = 8) -> Optional[OpResult]:
        """Collective second half: wait for the launched fills, report
        failures (re-filling from the re-picked source while allowed) and
        complete every shard.  One all-gather per round: every rank derives
        every replica's decision (final or retry) from the same gathered
        outcomes, so the loop ends everywhere together and the completions
        are applied in the same (rank) order on every registry replica."""
        txn = self._txn.pop(id(h), None) if h is not None else None
        active = bool(txn and txn["active"])
        result = txn["result"] if txn else None
        version = txn["version"] if txn else None
        loc = txn["loc"] if txn else []
        # a part that failed before launching (its bind) completes with the rest
        pending_done = None
        if h is not None and not active and result is not None and version is not None:
            pending_done = (h.model, h.replica, loc, int(result.status))
        rounds = 0
        done_by_rank = {}
        while True:
            outcome = None
            if active:
                n = h.num_shards
                sts, rsn = (C.c_int * n)(), (C.c_int * n)()
                step = lib.rs_transfer_wait if txn["launched"] else lib.rs_transfer_fill
                txn["launched"] = False
                step(h.h, C.cast(sts, C.c_void_p), C.cast(rsn, C.c_void_p))
                outcome = {"model": h.model, "replica": h.replica, "loc": loc,
                           "failed": {i: (int(sts[i]), int(rsn[i])) for i in loc if sts[i] != 0},
                           "src": self._source(h.model, h.replica)}
            elif pending_done is not None:
                outcome = {"done": pending_done}
                pending_done = None
            got = self.gather(outcome)
            reps = {}
            for o in got:
                if o is None or "done" in o:
                    continue
                st = reps.setdefault((o["model"], o["replica"]), {"failed": {}, "retry": True})
                for i, (code, reason) in o["failed"].items():
                    st["failed"][i] = code
                    st["retry"] &= self._apply(("report", o["model"], o["replica"], i, o["src"],
                                                reason)) == 0
            any_active = False
            for rk, o in enumerate(got):
                if o is None:
                    continue
                if "done" in o:
                    done_by_rank[rk] = o["done"]
                    continue
                st = reps[(o["model"], o["replica"])]
                if not st["failed"]:
                    fin = Status.ok
                elif not (st["retry"] and rounds + 1 < max_rounds):
                    fin = Status(next(iter(st["failed"].values())))
                else:
                    any_active = True  # this part refills from the re-picked source
                    continue
                done_by_rank[rk] = (o["model"], o["replica"], o["loc"], int(fin))
                if rk == self.rank:
                    lib.rs_transfer_finish(h.h, version, int(fin == Status.ok))
                    result = OpResult(fin, version if fin == Status.ok else None, txn["changed"])
                    active = False
            if not any_active:
                break
            rounds += 1
        for rk in sorted(done_by_rank):
            m, r, shards, st = done_by_rank[rk]
            for i in shards:
                self._apply(("complete", m, r, i, st))
        return result

    def update(self, h: Optional[Handle], spec: str = "latest") -> Optional[OpResult]:
        return self.replicate(h, spec, update=True)

    # ---- introspection (local registry replica) -----------------------------
    def assigns(self):
        return self.local.assigns()

    def listing(self, model="m"):
        return self.local.listing(model)
