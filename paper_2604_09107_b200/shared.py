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

A replica's shards may live in several member processes (a TP/FSDP group):
each process appends its shards' part of every replica operation and the
registry replicas apply the operation once all parts are in the log -- the
reference server's group transactions, with an abort entry for stragglers.
"""
from __future__ import annotations

import ctypes as C
import os
import threading
import time
import uuid
from typing import Optional

import msgpack

from ._lib import lib
from .dist import apply_op, lib_manifest
from .ros import Cluster, Handle, OpResult, Status, _read_bytes, check, combine_layout_key


def _b(s: str) -> bytes:
    return s.encode()


def _enc(origin: str, op: tuple) -> bytes:
    """A log entry: (origin, op) in msgpack -- plain data only (bytes, str,
    ints, bools, None, sequences, maps); nothing in an entry is executable,
    so a stray writer on the log port cannot run code in the members."""
    return msgpack.packb((origin, op), use_bin_type=True)


def _dec(entry: bytes):
    """(origin, op) with every sequence as a tuple (ops and transaction keys
    are tuples; keys must stay hashable)."""
    return msgpack.unpackb(entry, raw=False, use_list=False, strict_map_key=False)


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
        self._w3 = _Conn(host, port, timeout_s)  # appends of the seed-fill waiter
        self._seed = None
        self._r = _Conn(host, port, timeout_s)  # the follower's tail
        self._fin = None
        self._cv = threading.Condition()
        self.applied = 0
        self._rc = {}        # seq -> status code of this member's own ops
        self._txn = {}       # id(handle) -> (version, changed) between replicate_start/finish
        self._txns = {}      # group transactions (applied by the follower)
        self._ctr = {}       # (model, replica, kind) -> operations issued
        self._stop = False
        self._err = None
        self._t = threading.Thread(target=self._follow, daemon=True)
        self._t.start()

    # ---- the log ------------------------------------------------------------
    def _follow(self):
        try:
            while not self._stop:
                for e in self._r.fetch(self.applied, 50):
                    # an entry no member could have written (a stray or hostile
                    # writer) is skipped the same way by every replica
                    origin, rc = None, int(Status.protocol_error)
                    try:
                        origin, op = _dec(e)
                        if isinstance(op, tuple) and op and isinstance(op[0], str):
                            rc = self._apply(origin, op)
                    except Exception:  # noqa: BLE001 - malformed entry or operation
                        pass
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
        if kind == "part":
            return self._part(op)
        if kind == "txn_abort":
            t = self._txns.setdefault(op[1], {"n": 0, "parts": {}, "meta": {}, "state": "pending", "rc": None})
            if t["state"] == "pending":
                t["state"], t["rc"] = "aborted", int(Status.group_aborted)
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
        seq = self._w.append(_enc(self.me, o))
        if not self._wait(lambda: self.applied > seq):
            raise TimeoutError(f"op {o[0]} (seq {seq}) not applied")
        with self._cv:
            return self._rc.pop(seq, 0)

    def sync(self) -> None:
        """Catch up with every entry appended so far."""
        self.op(("noop",))

    def announce(self, blobs) -> None:
        if blobs:
            self._w.append(_enc(self.me, ("import", list(blobs))))

    def close(self):
        if self._fin is not None:
            self._fin.join(60)
        if self._seed is not None:
            self._seed.join(120)
        self._stop = True
        self._t.join(timeout=5)
        self._w3.close()
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

    # ---- group transactions ------------------------------------------------------
    # A replica's shards may live in several member processes (a TP/FSDP
    # group, one process per GPU).  Like the reference server joining
    # per-shard requests into one group transaction (txn_arrive /
    # maybe_start_txn, server_core.cpp:298-591), each member appends its
    # shards' part of a replica operation; every registry replica applies the
    # operation once the parts of all shards are in the log (the same entry
    # everywhere, so the same plan).  A member that waits too long appends
    # an abort; whichever of the last part or the abort comes first in the
    # log decides, and an aborted transaction answers group_aborted.  Members
    # of a replica issue its operations in the same order
    # (ClientConfig.first_shard/group_shards, config.hpp:28-33).
    def _txn_key(self, h: Handle, kind: str):
        k = (h.model, h.replica, kind)
        c = self._ctr.get(k, 0)
        self._ctr[k] = c + 1
        return (h.model, h.replica, kind, c)

    def _part(self, op) -> int:
        _, key, n, parts, meta = op
        t = self._txns.setdefault(key, {"n": n, "parts": {}, "meta": {}, "state": "pending", "rc": None})
        if t["state"] != "pending":
            return t["rc"] if t["state"] == "done" else int(Status.group_aborted)
        t["parts"].update(parts)
        for k, v in meta.items():  # per-member extras (retention lags, provisional)
            if isinstance(v, (list, tuple)):
                t["meta"][k] = sorted(set(t["meta"].get(k, [])) | set(v))
            elif isinstance(v, bool):
                t["meta"][k] = t["meta"].get(k, False) or v
            else:
                t["meta"][k] = v
        if sorted(t["parts"]) == list(range(n)):
            t["rc"] = self._start_txn(key, t)
            t["state"] = "done"
        return 0

    def _start_txn(self, key, t) -> int:
        m, r, kind = key[0], key[1], key[2]
        n, parts, meta = t["n"], t["parts"], t["meta"]
        c = self.local.h
        if kind == "open":
            eps = [parts[i]["ep"] for i in range(n)]
            lk = combine_layout_key([parts[i]["hash"] for i in range(n)])
            geo = any(parts[i]["hash"][1] for i in range(n))
            dman = [parts[i]["dm"] for i in range(n)] if geo else []
            dlay = [parts[i]["dl"] for i in range(n)] if geo else []
            rc = apply_op(c, ("open", m, r, n, meta["dc"], eps, lk, dman, dlay))
            if rc == 0 and meta.get("retain"):
                rc = apply_op(c, ("retain", m, r, list(meta["retain"])))
            if rc == 0 and meta.get("seed"):
                rc = apply_op(c, ("seed_on", m, r))
            return rc
        if kind == "publish":
            return apply_op(c, ("publish", m, r, meta["v"], [parts[i][0] for i in range(n)],
                                [parts[i][1] for i in range(n)], meta.get("prov", False)))
        if kind == "finalize":
            return apply_op(c, ("finalize", m, r, meta["v"], [parts[i] for i in range(n)]))
        if kind == "replicate":
            if meta["update"]:
                return apply_op(c, ("update", m, r, meta["spec"], meta["cur"]))
            return apply_op(c, ("replicate", m, r, meta["spec"]))
        if kind == "unpublish":
            return apply_op(c, ("unpublish", m, r))
        if kind == "close":
            return apply_op(c, ("close", m, r))
        raise ValueError(kind)

    def _group(self, h: Handle, kind: str, parts: dict, meta: dict, timeout: float = 120.0,
               key=None) -> int:
        """Appends this member's part of a replica operation; returns its
        status once the group transaction started (or group_aborted)."""
        return self.group_op(key or self._txn_key(h, kind), h.num_shards, parts, meta, timeout)

    def group_op(self, key, n: int, parts: dict, meta: dict, timeout: float = 120.0) -> int:
        """One member's part (shard -> payload) of the group transaction
        `key` = (model, replica, kind, k) over n shards."""
        self._w.append(_enc(self.me, ("part", key, n, parts, meta)))
        state = lambda: self._txns.get(key, {}).get("state")  # noqa: E731
        if not self._wait(lambda: state() in ("done", "aborted"), timeout):
            self._w.append(_enc(self.me, ("txn_abort", key)))
            self._wait(lambda: state() in ("done", "aborted"), timeout)
        with self._cv:
            t = self._txns[key]
            return int(t["rc"]) if t["state"] == "done" else int(Status.group_aborted)

    # ---- ops -------------------------------------------------------------------
    def create(self, model: str, replica: str, num_shards: int = 1, **cfg) -> Handle:
        """Local: a handle to register tensors on, before open()."""
        h = self.local.open(model, replica, num_shards, **cfg)
        h.offload_seed = bool(cfg.get("offload_seed", False))
        return h

    def open(self, h: Handle, endpoints=None, datacenter: str = "dc0", timeout: float = 120.0) -> None:
        """Announces the replica (ClientCore::open): endpoints, slicing key,
        derived manifests of a resharding replica, retention rule -- the
        shards this process holds; the replica opens once every shard's
        part is in."""
        loc = h.local_shards()
        if not loc:
            raise ValueError(f"{h.replica}: no shard registered in this process")
        if endpoints is None:
            eps = {s: f"{self.me}:{s}" for s in loc}
        elif isinstance(endpoints, dict):
            eps = dict(endpoints)
        else:
            eps = dict(zip(loc, endpoints))
        parts = {}
        for sh in loc:
            h.set_endpoint(sh, eps[sh])
            hs = h.shard_hash(sh)
            parts[sh] = {"ep": eps[sh], "hash": hs,
                         "dm": h.derived(sh, 0) if hs[1] else b"", "dl": h.derived(sh, 1) if hs[1] else b""}
        meta = {"dc": datacenter, "retain": list(getattr(h, "retain", []) or []),
                "seed": bool(getattr(h, "offload_seed", False))}
        rc = self._group(h, "open", parts, meta, timeout)
        if rc:
            raise RuntimeError(f"open {h.replica}: {Status(rc).name}")

    def publish(self, h: Handle, version: int, timeout: float = 120.0) -> OpResult:
        """publish() of this process's shards (a group transaction over the
        replica's shards).  With early_publish the provisional manifests go
        in at once and a background thread appends the final ones (a
        "finalize" transaction) when the big-entry digests are done."""
        check(lib.rs_prepare_publish(h.h, version), "rs_prepare_publish")
        loc = h.local_shards()
        early = h.publish_pending
        parts = {s: (lib_manifest(h, s), h.layout(s)) for s in loc}
        rc = self._group(h, "publish", parts, {"v": version, "prov": early}, timeout)
        lib.rs_commit_publish(h.h, version, rc)
        if rc == 0:
            self.announce([h.serve_export(s) for s in loc])
            if early:
                key = (h.model, h.replica, "finalize", version)

                def fin():
                    if lib.rs_publish_finalize(h.h, 60.0) == 0:
                        part = {s: h.manifest(s) for s in loc}
                        self._w2.append(_enc(self.me, ("part", key, h.num_shards, part,
                                                       {"v": version})))
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
        loc = h.local_shards()
        good = lib.rs_offload_lanes(h.h, v.value) == 0
        blobs = [_read_bytes(lib.rs_lane_export, h.h, s, v.value) for s in loc] if good else []
        self.announce(blobs)
        for s in loc:
            self.op(("offload_confirm", h.model, h.replica, s, v.value, good, f"host:{h.replica}:{s}"))

    def unpublish(self, h: Handle, timeout: float = 120.0) -> OpResult:
        self.finalized(h)  # an early publish's digests still read the regions
        rc = self._group(h, "unpublish", {s: None for s in h.local_shards()}, {}, timeout)
        self._offload_first(h)
        done, s, _, _ = self.result(h.model, h.replica)
        return OpResult(Status(rc) if rc else (s if done else Status.timeout))

    def replicate(self, h: Handle, spec: str = "latest", update: bool = False, wait_s: float = 60.0,
                  max_rounds: int = 8) -> OpResult:
        """ClientCore::replicate / update for this member's shards of the
        replica: plan (a group transaction through the log), bind and
        announce the serve state (downstream members may chase it at once),
        fill -- reporting failures through the log and refilling from the
        re-picked source -- and complete.  = replicate_start + replicate_finish."""
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
        loc = h.local_shards()
        rc = self._group(h, "replicate", {s: None for s in loc},
                         {"spec": spec, "update": update, "cur": cur}, wait_s)
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
            self._start_seed(h)
            return OpResult(Status.ok, v or cur, False)
        rc = lib.rs_transfer_bind(h.h, v)
        if rc:
            for i in loc:
                self.op(("complete", h.model, h.replica, i, rc))
            lib.rs_transfer_finish(h.h, v, 0)
            return OpResult(Status(rc))
        self.announce([h.serve_export(i) for i in loc])
        self._txn[id(h)] = (v, ch or not update)
        return None

    def replicate_finish(self, h: Handle, max_rounds: int = 8, wait_s: float = 120.0) -> OpResult:
        """Second half: fill this process's shards (launch + wait), failure
        reports, completion; the outcome is the replica's (all shards)."""
        v, changed = self._txn.pop(id(h))
        n = h.num_shards
        loc = h.local_shards()
        final = None
        for _ in range(max_rounds):
            sts, rsn = (C.c_int * n)(), (C.c_int * n)()
            lib.rs_transfer_fill(h.h, C.cast(sts, C.c_void_p), C.cast(rsn, C.c_void_p))
            failed = {i: (int(sts[i]), int(rsn[i])) for i in loc if sts[i] != 0}
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
        for i in loc:
            self.op(("complete", h.model, h.replica, i, int(final)))
        if final == Status.ok and len(loc) < n:
            # the replica is published only when every process's shards are
            self._wait(lambda: (self.local.view(h.model, h.replica) or {}).get("lifecycle") != "replicating",
                       wait_s)
            life = (self.local.view(h.model, h.replica) or {}).get("lifecycle")
            if life != "published":
                final = Status.transfer_failed
        lib.rs_transfer_finish(h.h, v, int(final == Status.ok))
        return OpResult(final, v if final == Status.ok else None, changed)

    # ---- cross-link seed buffers (client_core.cpp:1720-1812) -----------------
    def _start_seed(self, h: Handle) -> None:
        """An update without change whose outcome starts a seed fill: fill this
        member's shards into pinned host memory in the background; when done,
        announce the lanes (other members import them) and append the
        role-seed completions, so every registry replica publishes the seed."""
        from ._lib import RsAssignment
        a = RsAssignment()
        loc = h.local_shards()
        if not loc or lib.rs_server_seed_start(self.local.h, _b(h.model), _b(h.replica), loc[0],
                                               C.byref(a)) != 1:
            return
        v = a.version
        if self._seed is not None:
            self._seed.join()
        rc = lib.rs_seed_fill(h.h)

        def wait():
            lib.rs_seed_wait(h.h)
            sts = {s: (lib.rs_seed_status(h.h, s) if rc == 0 else rc) for s in loc}
            blobs = [_read_bytes(lib.rs_seed_export, h.h, s, v) for s in loc if sts[s] == 0]
            if blobs:
                self._w3.append(_enc(self.me, ("import", blobs)))
            for s in loc:
                self._w3.append(_enc(self.me, ("seed_complete", h.model, h.replica, s,
                                               int(sts[s]), v)))
        self._seed = threading.Thread(target=wait, daemon=True)
        self._seed.start()

    def seed_wait(self, h: Handle, timeout: float = 120.0) -> None:
        """Wait until this member's seed fill is reported to the log."""
        if self._seed is not None:
            self._seed.join(timeout)
            self._seed = None
        self.sync()

    def update(self, h: Handle, spec: str = "latest", wait_s: float = 60.0) -> OpResult:
        return self.replicate(h, spec, update=True, wait_s=wait_s)

    def leave(self, h: Handle) -> None:
        """ClientCore::close: the replica leaves the deployment (once every
        process holding its shards left)."""
        self._group(h, "close", {s: None for s in h.local_shards()}, {})
        h.close()
