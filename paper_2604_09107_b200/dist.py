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
from .ros import Cluster, Handle, OpResult, Status, _read_bytes, check


def _b(s: str) -> bytes:
    return s.encode()


def _blob_arrays(blobs):
    arr = (C.c_char_p * max(len(blobs), 1))(*blobs)
    lens = (C.c_size_t * max(len(blobs), 1))(*[len(x) for x in blobs])
    return C.cast(arr, C.c_void_p), C.cast(lens, C.c_void_p), arr, lens


class DistCluster:
    def __init__(self, group=None, pipeline: bool = True, smart_skipping: bool = True):
        import torch.distributed as dist
        self.dist = dist
        self.rank = dist.get_rank()
        self.world = dist.get_world_size()
        self.pg = group if group is not None else dist.new_group(backend="gloo")
        self.local = Cluster(pipeline=pipeline, smart_skipping=smart_skipping)

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
        c = self.local.h
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
            pm, pl, _k1, _k2 = _blob_arrays(mans)
            if lays:
                qm, ql, _k3, _k4 = _blob_arrays(lays)
            else:
                qm = ql = None
            return lib.rs_server_publish(c, _b(m), _b(r), v, len(mans), pm, pl, qm, ql)
        if kind == "add_layout":
            _, m, v, key, mans, lays = o
            pm, pl, _k1, _k2 = _blob_arrays(mans)
            qm, ql, _k3, _k4 = _blob_arrays(lays)
            return lib.rs_server_add_layout(c, _b(m), v, _b(key), len(mans), pm, pl, qm, ql)
        if kind == "unpublish":
            return lib.rs_server_unpublish(c, _b(o[1]), _b(o[2]))
        if kind == "replicate":
            return lib.rs_server_replicate(c, _b(o[1]), _b(o[2]), _b(o[3]))
        if kind == "update":
            _, m, r, sp, cur = o
            return lib.rs_server_update(c, _b(m), _b(r), _b(sp), int(cur is not None), cur or 0)
        if kind == "complete":
            return lib.rs_server_complete(c, _b(o[1]), _b(o[2]), o[3], o[4])
        if kind == "report":
            return lib.rs_server_failure_report(c, _b(o[1]), _b(o[2]), o[3], _b(o[4]), o[5])
        raise ValueError(kind)

    def result(self, model, replica):
        d, s, v, ch = C.c_int(), C.c_int(), C.c_uint64(), C.c_int()
        lib.rs_server_result(self.local.h, _b(model), _b(replica), C.byref(d), C.byref(s),
                             C.byref(v), C.byref(ch))
        return bool(d.value), Status(s.value), v.value, bool(ch.value)

    # ---- ops ---------------------------------------------------------------
    def create(self, model: str, replica: str, num_shards: int = 1, **cfg) -> Handle:
        """Local: a handle to register tensors on, before the collective open()."""
        return self.local.open(model, replica, num_shards, **cfg)

    def open(self, h: Optional[Handle], endpoints: Optional[list[str]] = None,
             datacenter: str = "dc0") -> None:
        """Collective: every rank mirrors every opened replica's record
        (with its slicing key, known once its tensors are registered)."""
        mine = None
        if h is not None:
            eps = endpoints or [f"rank{self.rank}:{i}" for i in range(h.num_shards)]
            for i, e in enumerate(eps):
                h.set_endpoint(i, e)
            key = h.layout_key
            dman = [h.derived(s, 0) for s in range(h.num_shards)] if key else []
            dlay = [h.derived(s, 1) for s in range(h.num_shards)] if key else []
            mine = ("open", h.model, h.replica, h.num_shards, datacenter, eps, key, dman, dlay)
        for rc in self.server_ops(mine):
            assert rc in (None, 0), rc

    def publish(self, h: Optional[Handle], version: int) -> Optional[OpResult]:
        mine = None
        if h is not None:
            check(lib.rs_prepare_publish(h.h, version), "rs_prepare_publish")
            mine = ("publish", h.model, h.replica, version,
                    [h.manifest(s) for s in range(h.num_shards)],
                    [h.layout(s) for s in range(h.num_shards)])
        rcs = self.server_ops(mine)
        blobs = None
        if h is not None:
            st = rcs[self.rank]
            lib.rs_commit_publish(h.h, version, st)
            if st == 0:
                blobs = [h.serve_export(s) for s in range(h.num_shards)]
        self._import_all(self.gather(blobs))
        if h is None:
            return None
        st = Status(rcs[self.rank])
        return OpResult(st, version if st == Status.ok else None)

    def unpublish(self, h: Optional[Handle]) -> Optional[OpResult]:
        rcs = self.server_ops(("unpublish", h.model, h.replica) if h is not None else None)
        if h is None:
            return None
        done, s, _, _ = self.result(h.model, h.replica)
        st = Status(rcs[self.rank]) if rcs[self.rank] else s
        return OpResult(st if done else Status.timeout)

    def replicate(self, h: Optional[Handle], spec: str = "latest", update: bool = False,
                  max_rounds: int = 8) -> Optional[OpResult]:
        """Collective replicate/update: plan on every rank, bind + serve,
        exchange serve states, then every reader fills (kernels chase each
        other's watermarks), with failure reports applied collectively."""
        mine = None
        if h is not None:
            cur = h.current_version
            mine = ("update", h.model, h.replica, spec, cur) if update else \
                ("replicate", h.model, h.replica, spec)
        self.server_ops(mine)
        active, result, version, changed = False, None, None, False
        if h is not None:
            d, s, v, ch = self.result(h.model, h.replica)
            if not d:
                result = OpResult(Status.timeout)  # parked: no version yet
            elif s != Status.ok:
                result = OpResult(s)
            elif update and not ch:
                result = OpResult(Status.ok, v or cur, False)
            else:
                version, changed = v, ch or not update
                rc = lib.rs_transfer_bind(h.h, version)
                if rc != 0:
                    result = OpResult(Status(rc))
                else:
                    active = True
        blobs = [h.serve_export(s) for s in range(h.num_shards)] if active else None
        self._import_all(self.gather(blobs))
        rounds = 0
        while True:
            outcome = None
            if active:
                n = h.num_shards
                sts, rsn = (C.c_int * n)(), (C.c_int * n)()
                lib.rs_transfer_fill(h.h, C.cast(sts, C.c_void_p), C.cast(rsn, C.c_void_p))
                outcome = (h.model, h.replica, [int(x) for x in sts], [int(x) for x in rsn],
                           self._source(h.model, h.replica))
            retry = {}
            for o in self.gather(outcome):
                if o is None:
                    continue
                m, r, sts, rsn, src = o
                failed = [i for i, x in enumerate(sts) if x != 0]
                if not failed:
                    continue
                good = True
                for i in failed:
                    good &= self._apply(("report", m, r, i, src, rsn[i])) == 0
                retry[r] = good and rounds + 1 < max_rounds
            if active:
                mine_failed = any(x != 0 for x in outcome[2])
                if not mine_failed or not retry.get(h.replica, False):
                    if mine_failed:
                        result = OpResult(Status(next(x for x in outcome[2] if x != 0)))
                        lib.rs_transfer_finish(h.h, version, 0)
                    else:
                        lib.rs_transfer_finish(h.h, version, 1)
                        result = OpResult(Status.ok, version, changed)
                    active = False
            if not any(self.gather(active)):
                break
            rounds += 1
        done = (h.model, h.replica, h.num_shards, int(result.status)) if (
            h is not None and result is not None and version is not None) else None
        for o in self.gather(done):
            if o is None:
                continue
            m, r, n, st = o
            for i in range(n):
                self._apply(("complete", m, r, i, st))
        return result

    def update(self, h: Optional[Handle], spec: str = "latest") -> Optional[OpResult]:
        return self.replicate(h, spec, update=True)

    # ---- introspection (local registry replica) -----------------------------
    def assigns(self):
        return self.local.assigns()

    def listing(self, model="m"):
        return self.local.listing(model)
