"""Dynamic membership: processes join and leave a deployment at any time.

The reference has one metadata server that clients dial whenever they start
(ServerCore behind StreamServerHost; StreamControl, transport_stream.cpp:
582-797).  Here every process holds a replica of the registry
(csrc/registry.cpp) and the replicas follow one totally ordered operation log
(csrc/oplog.cpp, a replicated state machine):

* ``LogServer`` hosts the log (any process, or a standalone one);
* ``SharedCluster`` is one process's member: a follower thread tails the log
  and applies every entry, in order, to the local registry replica -- and
  imports the serve states (CUDA IPC handles) other members announce, so this
  process's readers can pull from, and chase, replicas living elsewhere;
* a process's own operation is appended to the log and takes effect when the
  follower reaches it, so every replica sees the same request sequence and
  computes the same plan (the reference SimExecutor order for simultaneous
  readers: a chain).

A process that starts late replays the log from entry 0: it joins with the
registry state everyone else has, including replicas that are still filling,
so it can be planned onto a partially landed copy (config 4's elastic join).
No collective and no fixed process group: unlike ``dist.DistCluster`` (the
lock-step gloo variant), nobody waits for a member that is not there.

Every replica a SharedCluster opens must have all its shards in this process
(a TP/FSDP group spread over processes uses ``dist.DistCluster``).
"""
from __future__ import annotations

import ctypes as C
import os
import pickle
import threading
import time
import uuid
from typing import Optional

from ._lib import lib
from .dist import apply_op, lib_manifest
from .ros import Cluster, Handle, OpResult, Status, _read_bytes, check, combine_layout_key


def _b(s: str) -> bytes:
    return s.encode()


class LogServer:
    """Hosts the registry's operation log (rs_oplog_serve)."""

    def __init__(self, host: str = "127.0.0.1", port: int = 0):
        self.h = C.c_void_p()
        p = C.c_int()
        check(lib.rs_oplog_serve(_b(host), port, C.byref(p), C.byref(self.h)), "rs_oplog_serve")
        self.host, self.port = host, p.value

    @property
    def size(self) -> int:
        return int(lib.rs_oplog_server_size(self.h))

    def close(self):
        if self.h:
            lib.rs_oplog_server_stop(self.h)
            self.h = None


class _Conn:
    def __init__(self, host, port, timeout_s):
        self.h = C.c_void_p()
        check(lib.rs_oplog_connect(_b(host), port, timeout_s, C.byref(self.h)), "rs_oplog_connect")

    def append(self, entry: bytes) -> int:
        seq = C.c_uint64()
        check(lib.rs_oplog_append(self.h, entry, len(entry), C.byref(seq)), "rs_oplog_append")
        return seq.value

    def fetch(self, start: int, wait_ms: int, max_entries: int = 256) -> list[bytes]:
        n = C.c_uint64()
        check(lib.rs_oplog_fetch(self.h, start, wait_ms, max_entries, C.byref(n)), "rs_oplog_fetch")
        out = []
        for i in range(n.value):
            p, ln = C.c_void_p(), C.c_size_t()
            check(lib.rs_oplog_entry(self.h, i, C.byref(p), C.byref(ln)))
            out.append(C.string_at(p, ln.value))
        return out

    def close(self):
        if self.h:
            lib.rs_oplog_close(self.h)
            self.h = None


class SharedCluster:
    """This process's member of a deployment whose registry replicas follow
    one operation log.  Every method acts for this process only (no
    collective)."""

    def __init__(self, host: str, port: int, pipeline: bool = True, smart_skipping: bool = True,
                 timeout_s: float = 10.0):
        self.local = Cluster(pipeline=pipeline, smart_skipping=smart_skipping)
        self.me = f"{os.getpid()}-{uuid.uuid4().hex[:8]}"
        self._w = _Conn(host, port, timeout_s)  # appends (caller's thread)
        self._w2 = _Conn(host, port, timeout_s)  # appends of the early-publish finalizer
        self._r = _Conn(host, port, timeout_s)  # the follower's tail
        self._fin = None
        self._cv = threading.Condition()
        self.applied = 0
        self._rc = {}        # seq -> status code of this member's own ops
        self._txn = {}       # id(handle) -> (version, changed) between replicate_start/finish
        self._stop = False
        self._err = None
        self._t = threading.Thread(target=self._follow, daemon=True)
        self._t.start()

    # ---- the log ------------------------------------------------------------
    def _follow(self):
        try:
            while not self._stop:
                for e in self._r.fetch(self.applied, 50):
                    origin, op = pickle.loads(e)
                    rc = self._apply(origin, op)
                    with self._cv:
                        if origin == self.me:
                            self._rc[self.applied] = rc
                        self.applied += 1
                        self._cv.notify_all()
        except Exception as ex:  # noqa: BLE001 - surfaced to the caller's waits
            if not self._stop:
                with self._cv:
                    self._err = ex
                    self._cv.notify_all()

    def _apply(self, origin, op) -> int:
        kind = op[0]
        if kind == "noop":
            return 0
        if kind == "import":  # serve states another member announces
            if origin != self.me:
                for b in op[1]:
                    lib.rs_serve_import(self.local.h, b, len(b))
            return 0
        return apply_op(self.local.h, op)

    def _wait(self, pred, timeout: float = 60.0):
        deadline = time.time() + timeout
        with self._cv:
            while not pred():
                if self._err is not None:
                    raise RuntimeError(f"op log follower failed: {self._err!r}")
                left = deadline - time.time()
                if left <= 0:
                    return False
                self._cv.wait(left)
        return True

    def op(self, o) -> int:
        """Appends one registry operation; returns its status once this
        member's replica has applied it (with everything sequenced before)."""
        seq = self._w.append(pickle.dumps((self.me, o)))
        if not self._wait(lambda: self.applied > seq):
            raise TimeoutError(f"op {o[0]} (seq {seq}) not applied")
        with self._cv:
            return self._rc.pop(seq, 0)

    def sync(self) -> None:
        """Catch up with every entry appended so far."""
        self.op(("noop",))

    def announce(self, blobs) -> None:
        if blobs:
            self._w.append(pickle.dumps((self.me, ("import", list(blobs)))))

    def close(self):
        if self._fin is not None:
            self._fin.join(60)
        self._stop = True
        self._t.join(timeout=5)
        self._w2.close()
        self._w.close()
        self._r.close()
        self.local.close()

    # ---- registry views (this member's replica) ------------------------------
    def result(self, model, replica):
        d, s, v, ch = C.c_int(), C.c_int(), C.c_uint64(), C.c_int()
        lib.rs_server_result(self.local.h, _b(model), _b(replica), C.byref(d), C.byref(s), C.byref(v),
                             C.byref(ch))
        return bool(d.value), Status(s.value), v.value, bool(ch.value)

    def assigns(self):
        return self.local.assigns()

    def listing(self, model="m"):
        return self.local.listing(model)

    def _source(self, model, replica) -> str:
        return _read_bytes(lib.rs_cluster_source, self.local.h, _b(model), _b(replica)).decode()

    # ---- ops -------------------------------------------------------------------
    def create(self, model: str, replica: str, num_shards: int = 1, **cfg) -> Handle:
        """Local: a handle to register tensors on, before open()."""
        return self.local.open(model, replica, num_shards, **cfg)

    def open(self, h: Handle, endpoints=None, datacenter: str = "dc0") -> None:
        """Announces the replica (ClientCore::open): endpoints, slicing key,
        derived manifests of a resharding replica, retention rule."""
        n = h.num_shards
        if h.local_shards() != list(range(n)):
            raise ValueError(f"{h.replica}: every shard must be registered in this process")
        eps = list(endpoints) if endpoints is not None else [f"{self.me}:{s}" for s in range(n)]
        for s, e in enumerate(eps):
            h.set_endpoint(s, e)
        hashes = [h.shard_hash(s) for s in range(n)]
        key = combine_layout_key(hashes)
        geo = any(x[1] for x in hashes)
        dman = [h.derived(s, 0) for s in range(n)] if geo else []
        dlay = [h.derived(s, 1) for s in range(n)] if geo else []
        rc = self.op(("open", h.model, h.replica, n, datacenter, eps, key, dman, dlay))
        if rc:
            raise RuntimeError(f"open {h.replica}: {Status(rc).name}")
        if getattr(h, "retain", None):
            self.op(("retain", h.model, h.replica, list(h.retain)))

    def publish(self, h: Handle, version: int) -> OpResult:
        """publish(); with early_publish the provisional manifests go in at
        once and a background thread appends the final ones ("finalize")
        when the big-entry digests are done."""
        check(lib.rs_prepare_publish(h.h, version), "rs_prepare_publish")
        n = h.num_shards
        early = h.publish_pending
        rc = self.op(("publish", h.model, h.replica, version, [lib_manifest(h, s) for s in range(n)],
                      [h.layout(s) for s in range(n)], early))
        lib.rs_commit_publish(h.h, version, rc)
        if rc == 0:
            self.announce([h.serve_export(s) for s in range(n)])
            if early:
                def fin():
                    if lib.rs_publish_finalize(h.h, 60.0) == 0:
                        self._w2.append(pickle.dumps((self.me, ("finalize", h.model, h.replica, version,
                                                                [h.manifest(s) for s in range(n)]))))
                self._fin = threading.Thread(target=fin, daemon=True)
                self._fin.start()
        st = Status(rc)
        return OpResult(st, version if st == Status.ok else None)

    def finalized(self, h: Handle, timeout: float = 60.0) -> None:
        """Wait until an early publish's final manifests are in the log."""
        if self._fin is not None:
            self._fin.join(timeout)
            self._fin = None

    def _offload_first(self, h: Handle) -> None:
        v = C.c_uint64()
        if not lib.rs_server_offload_pending(self.local.h, _b(h.model), _b(h.replica), C.byref(v)):
            return
        good = lib.rs_offload_lanes(h.h, v.value) == 0
        blobs = [_read_bytes(lib.rs_lane_export, h.h, s, v.value) for s in range(h.num_shards)] if good else []
        self.announce(blobs)
        for s in range(h.num_shards):
            self.op(("offload_confirm", h.model, h.replica, s, v.value, good, f"host:{h.replica}:{s}"))

    def unpublish(self, h: Handle) -> OpResult:
        self.finalized(h)  # an early publish's digests still read the regions
        rc = self.op(("unpublish", h.model, h.replica))
        self._offload_first(h)
        done, s, _, _ = self.result(h.model, h.replica)
        return OpResult(Status(rc) if rc else (s if done else Status.timeout))

    def replicate(self, h: Handle, spec: str = "latest", update: bool = False, wait_s: float = 60.0,
                  max_rounds: int = 8) -> OpResult:
        """ClientCore::replicate / update for this member's replica: plan
        (through the log), bind and announce the serve state (downstream
        members may chase it at once), fill -- reporting failures through the
        log and refilling from the re-picked source -- and complete.
        = replicate_start + replicate_finish."""
        early = self.replicate_start(h, spec, update, wait_s)
        if early is not None:
            return early
        return self.replicate_finish(h, max_rounds)

    def replicate_start(self, h: Handle, spec: str = "latest", update: bool = False,
                        wait_s: float = 60.0) -> Optional[OpResult]:
        """First half: plan, bind, announce the (empty) fill's serve state.
        Returns the outcome when there is nothing to fill (failure, parked
        timeout, update without change), else None: call replicate_finish."""
        cur = h.current_version
        rc = self.op(("update", h.model, h.replica, spec, cur) if update else
                     ("replicate", h.model, h.replica, spec))
        if rc:
            return OpResult(Status(rc))
        self._offload_first(h)
        # a parked replicate completes when a later entry (a publish) wakes it
        if not self._wait(lambda: self.result(h.model, h.replica)[0], wait_s):
            return OpResult(Status.timeout)
        _, s, v, ch = self.result(h.model, h.replica)
        if s != Status.ok:
            return OpResult(s)
        if update and not ch:
            return OpResult(Status.ok, v or cur, False)
        n = h.num_shards
        rc = lib.rs_transfer_bind(h.h, v)
        if rc:
            for i in range(n):
                self.op(("complete", h.model, h.replica, i, rc))
            lib.rs_transfer_finish(h.h, v, 0)
            return OpResult(Status(rc))
        self.announce([h.serve_export(i) for i in range(n)])
        self._txn[id(h)] = (v, ch or not update)
        return None

    def replicate_finish(self, h: Handle, max_rounds: int = 8) -> OpResult:
        """Second half: fill (launch + wait), failure reports, completion."""
        v, changed = self._txn.pop(id(h))
        n = h.num_shards
        final = None
        for _ in range(max_rounds):
            sts, rsn = (C.c_int * n)(), (C.c_int * n)()
            lib.rs_transfer_fill(h.h, C.cast(sts, C.c_void_p), C.cast(rsn, C.c_void_p))
            failed = {i: (int(sts[i]), int(rsn[i])) for i in range(n) if sts[i] != 0}
            if not failed:
                final = Status.ok
                break
            src = self._source(h.model, h.replica)
            retry = True
            for i, (code, reason) in failed.items():
                retry &= self.op(("report", h.model, h.replica, i, src, reason)) == 0
            if not retry:
                final = Status(next(iter(failed.values()))[0])
                break
        if final is None:
            final = Status.transfer_failed
        lib.rs_transfer_finish(h.h, v, int(final == Status.ok))
        for i in range(n):
            self.op(("complete", h.model, h.replica, i, int(final)))
        return OpResult(final, v if final == Status.ok else None, changed)

    def update(self, h: Handle, spec: str = "latest", wait_s: float = 60.0) -> OpResult:
        return self.replicate(h, spec, update=True, wait_s=wait_s)

    def leave(self, h: Handle) -> None:
        """ClientCore::close: the replica leaves the deployment."""
        self.op(("close", h.model, h.replica))
        h.close()
