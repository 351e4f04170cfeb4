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

All methods are collective over the group: every rank calls them in the
same order, passing its local handle (or None when it has no part in that
operation).
"""
from __future__ import annotations

import ctypes as C
from typing import Optional

from ._lib import lib
from .ros import Cluster, Handle, OpResult, Status, _read_bytes, check


def _b(s: str) -> bytes:
    return s.encode()


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

    def server_ops(self, op):
        """Collective: all-gather one registry operation per rank (or None)
        and apply them to the local registry replica in rank order.  Ops:
        ("open", model, replica, shards, dc, endpoints),
        ("publish", model, replica, version, [manifest bytes per shard]),
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
            _, m, r, n, dc, eps = o
            arr = (C.c_char_p * n)(*[_b(e) for e in eps])
            return lib.rs_server_open(c, _b(m), _b(r), n, _b(dc), C.cast(arr, C.c_void_p))
        if kind == "publish":
            _, m, r, v, mans = o
            arr = (C.c_char_p * len(mans))(*mans)
            lens = (C.c_size_t * len(mans))(*[len(x) for x in mans])
            return lib.rs_server_publish(c, _b(m), _b(r), v, len(mans), C.cast(arr, C.c_void_p),
                                         C.cast(lens, C.c_void_p))
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

    def _source(self, model, replica) -> str:
        return _read_bytes(lib.rs_cluster_source, self.local.h, _b(model), _b(replica)).decode()

    # ---- ops ---------------------------------------------------------------
    def open(self, model: str, replica: Optional[str], num_shards: int = 1,
             endpoints: Optional[list[str]] = None, datacenter: str = "dc0",
             **cfg) -> Optional[Handle]:
        """Collective open.  Ranks with replica=None only mirror the others'
        records.  Tensors are registered on the returned handle afterwards."""
        mine = None
        h = None
        if replica is not None:
            h = self.local.open(model, replica, num_shards, datacenter=datacenter, **cfg)
            eps = endpoints or [f"rank{self.rank}:{i}" for i in range(num_shards)]
            for i, e in enumerate(eps):
                h.set_endpoint(i, e)
            mine = (model, replica, num_shards, datacenter, eps)
        for op in self.gather(mine):
            if op is None:
                continue
            m, r, n, dc, eps = op
            arr = (C.c_char_p * n)(*[_b(e) for e in eps])
            check(lib.rs_server_open(self.local.h, _b(m), _b(r), n, _b(dc), C.cast(arr, C.c_void_p)),
                  "rs_server_open")
        return h

    def publish(self, h: Optional[Handle], version: int) -> Optional[OpResult]:
        mine = None
        if h is not None:
            check(lib.rs_prepare_publish(h.h, version), "rs_prepare_publish")
            mine = (h.model, h.replica, version, [h.manifest(s) for s in range(h.num_shards)])
        statuses = {}
        for op in self.gather(mine):
            if op is None:
                continue
            m, r, v, mans = op
            arr = (C.c_char_p * len(mans))(*mans)
            lens = (C.c_size_t * len(mans))(*[len(x) for x in mans])
            statuses[r] = lib.rs_server_publish(self.local.h, _b(m), _b(r), v, len(mans),
                                                C.cast(arr, C.c_void_p), C.cast(lens, C.c_void_p))
        blobs = None
        if h is not None:
            st = statuses[h.replica]
            lib.rs_commit_publish(h.h, version, st)
            if st == 0:
                blobs = [h.serve_export(s) for s in range(h.num_shards)]
        self._import_all(self.gather(blobs))
        if h is None:
            return None
        st = Status(statuses[h.replica])
        return OpResult(st, version if st == Status.ok else None)

    def unpublish(self, h: Optional[Handle]) -> Optional[OpResult]:
        mine = (h.model, h.replica) if h is not None else None
        res = {}
        for op in self.gather(mine):
            if op is not None:
                res[op[1]] = lib.rs_server_unpublish(self.local.h, _b(op[0]), _b(op[1]))
        if h is None:
            return None
        d, s, v, ch = C.c_int(), C.c_int(), C.c_uint64(), C.c_int()
        lib.rs_server_result(self.local.h, _b(h.model), _b(h.replica), C.byref(d), C.byref(s),
                             C.byref(v), C.byref(ch))
        st = Status(res[h.replica]) if res[h.replica] else Status(s.value)
        if not d.value:
            st = Status.timeout  # readers still draining
        return OpResult(st)

    def replicate(self, h: Optional[Handle], spec: str = "latest", update: bool = False,
                  max_rounds: int = 8) -> Optional[OpResult]:
        """Collective replicate/update: plan on every rank, bind + serve,
        exchange serve states, then every reader fills (kernels chase each
        other's watermarks), with failure reports applied collectively."""
        mine = None
        if h is not None:
            cur = h.current_version
            mine = (h.model, h.replica, spec, update, cur)
        for op in self.gather(mine):
            if op is None:
                continue
            m, r, sp, upd, cur = op
            if upd:
                lib.rs_server_update(self.local.h, _b(m), _b(r), _b(sp), int(cur is not None),
                                     cur or 0)
            else:
                lib.rs_server_replicate(self.local.h, _b(m), _b(r), _b(sp))
        # every rank: outcome of the local op
        active, result, version, changed = False, None, None, False
        if h is not None:
            d, s, v, ch = C.c_int(), C.c_int(), C.c_uint64(), C.c_int()
            lib.rs_server_result(self.local.h, _b(h.model), _b(h.replica), C.byref(d), C.byref(s),
                                 C.byref(v), C.byref(ch))
            if not d.value:
                result = OpResult(Status.timeout)  # parked: no version yet
            elif s.value != 0:
                result = OpResult(Status(s.value))
            elif update and not ch.value:
                result = OpResult(Status.ok, v.value or cur, False)
            else:
                version, changed = v.value, bool(ch.value) or not update
                rc = lib.rs_transfer_bind(h.h, version)
                if rc != 0:
                    result = OpResult(Status(rc))
                else:
                    active = True
        blobs = [h.serve_export(s) for s in range(h.num_shards)] if active else None
        self._import_all(self.gather(blobs))
        # fill rounds: failures are reported to every registry replica
        rounds = 0
        while True:
            outcome = None
            if active:
                n = h.num_shards
                sts, rsn = (C.c_int * n)(), (C.c_int * n)()
                lib.rs_transfer_fill(h.h, C.cast(sts, C.c_void_p), C.cast(rsn, C.c_void_p))
                srcs = self._source(h.model, h.replica)
                outcome = (h.model, h.replica, [int(x) for x in sts], [int(x) for x in rsn], srcs)
            outs = self.gather(outcome)
            retry = {}
            for o in outs:
                if o is None:
                    continue
                m, r, sts, rsn, src = o
                failed = [i for i, x in enumerate(sts) if x != 0]
                if not failed:
                    continue
                ok = True
                for i in failed:
                    rc = lib.rs_server_failure_report(self.local.h, _b(m), _b(r), i, _b(src), rsn[i])
                    ok &= rc == 0
                retry[r] = ok and rounds + 1 < max_rounds
            if active:
                mine_failed = any(x != 0 for x in outcome[2])
                if not mine_failed or not retry.get(h.replica, False):
                    if mine_failed:
                        bad = next(x for x in outcome[2] if x != 0)
                        result = OpResult(Status(bad))
                        lib.rs_transfer_finish(h.h, version, 0)
                    else:
                        lib.rs_transfer_finish(h.h, version, 1)
                        result = OpResult(Status.ok, version, changed)
                    active = False
            # the loop ends when no rank still has a retry pending
            if not any(self.gather(active)):
                break
            rounds += 1
        # completions, applied in rank order everywhere
        done = (h.model, h.replica, h.num_shards, int(result.status)) if (
            h is not None and result is not None and version is not None) else None
        for o in self.gather(done):
            if o is None:
                continue
            m, r, n, st = o
            for i in range(n):
                lib.rs_server_complete(self.local.h, _b(m), _b(r), i, st)
        return result

    def update(self, h: Optional[Handle], spec: str = "latest") -> Optional[OpResult]:
        return self.replicate(h, spec, update=True)

    # ---- introspection (local registry replica) -----------------------------
    def assigns(self):
        return self.local.assigns()

    def listing(self, model="m"):
        return self.local.listing(model)
