"""Python host mirror of the ROS API over the C ABI (include/ros_b200.h).

Names, argument meaning and status values follow the reference ClientCore /
ServerCore (/root/reference/proj/include/refstore/client_core.hpp:63-93,
server_core.hpp:37-52) so tests read like the reference's own
(tests/unit/test_client_core.cpp).  Two deployments:

* ``Cluster`` -- one process: a registry ("server A") shared by any number of
  handles, which may sit on different GPUs (peer access over NVLink).
* ``DistCluster`` -- one process per GPU (torchrun): every rank holds a
  replica of the registry and applies the same operation log in the same
  order (a replicated state machine over ``torch.distributed``), so every
  rank computes the same plan; serve states cross processes as CUDA IPC
  handles.  No NCCL collective touches the data path.
"""
from __future__ import annotations

import ctypes as C
import enum
import re
from dataclasses import dataclass, field
from typing import Optional

from ._lib import RsAssignment, RsConfig, RsStats, lib


class Status(enum.IntEnum):
    """refstore::Status (types.hpp:22-41)."""
    ok = 0
    invalid_argument = 1
    invalid_state = 2
    already_exists = 3
    not_found = 4
    version_regression = 5
    manifest_conflict = 6
    mutability_violation = 7
    version_unavailable = 8
    group_aborted = 9
    server_unavailable = 10
    transfer_failed = 11
    checksum_mismatch = 12
    not_serving = 13
    timeout = 14
    offload_failed = 15
    protocol_error = 16
    closed = 17


class ROSError(RuntimeError):
    def __init__(self, status: int, what: str = ""):
        self.status = Status(status)
        super().__init__(f"{what}: {self.status.name}" if what else self.status.name)


def check(rc: int, what: str = "") -> None:
    if rc != 0:
        raise ROSError(rc, what)


@dataclass
class OpResult:
    """ClientCore::OpResult (client_core.hpp:37-42)."""
    status: Status
    version: Optional[int] = None
    changed: bool = False


@dataclass
class Stats:
    bytes_pulled: int = 0
    bytes_pulled_cross_dc: int = 0
    bytes_copied_local: int = 0
    items_verified: int = 0
    checksum_failures: int = 0
    failure_reports: int = 0
    failovers: int = 0
    last_pull_ms: float = 0.0
    last_publish_ms: float = 0.0
    last_pull_bytes: int = 0
    last_pull_launches: int = 0
    h2d_bytes: int = 0
    d2h_bytes: int = 0
    fill_max_ms: float = 0.0
    fill_sum_ms: float = 0.0
    fill_bytes: int = 0
    kernel_launches: int = 0


@dataclass
class Assign:
    replica: str
    version: int
    src: str
    src_serving: int


def _b(s: str) -> bytes:
    return s.encode()


def _read_bytes(fn, *args) -> bytes:
    n = C.c_size_t(0)
    check(fn(*args, None, 0, C.byref(n)))
    buf = C.create_string_buffer(max(n.value, 1))
    check(fn(*args, buf, n.value, C.byref(n)))
    return buf.raw[:n.value]


def make_config(chunk_bytes=4096, tiny_threshold=2 << 20, group_target=64 << 20, pipeline=True,
                checksum_retries=3, pull_timeout_s=4.0, datacenter="dc0",
                reshard_align=2, grid_sms=0, early_publish=False, offload_seed=False) -> RsConfig:
    cfg = RsConfig()
    lib.rs_config_default(C.byref(cfg))
    cfg.chunk_bytes = chunk_bytes
    cfg.tiny_threshold = tiny_threshold
    cfg.group_target = group_target
    cfg.pipeline = int(pipeline)
    cfg.checksum_retries = checksum_retries
    cfg.pull_timeout_s = pull_timeout_s
    cfg.datacenter = datacenter.encode()
    cfg.reshard_align = reshard_align
    cfg.grid_sms = grid_sms
    cfg.early_publish = int(early_publish)
    cfg.offload_seed = int(offload_seed)
    return cfg


def tp_slice(shape, elem_bytes: int, split_dim, tp: int, rank: int):
    """Geometry (rows, row_bytes, r0, nr, c0, nc) of rank `rank`'s slice of a
    tensor of `shape` split `tp` ways along `split_dim` (None: replicated).
    1-D tensors are [1 x N]: a dim-0 split of them is a column split."""
    if len(shape) == 1:
        rows, w = 1, shape[0] * elem_bytes
        if split_dim is None or tp == 1:
            return rows, w, 0, 1, 0, w
        return rows, w, 0, 1, rank * w // tp, w // tp
    rows = shape[0]
    w = elem_bytes
    for d in shape[1:]:
        w *= d
    if split_dim is None or tp == 1:
        return rows, w, 0, rows, 0, w
    if split_dim == 0:
        return rows, w, rank * rows // tp, rows // tp, 0, w
    return rows, w, 0, rows, rank * w // tp, w // tp


_ASSIGN = re.compile(r"^\d+ assign (.*)$")


class Cluster:
    """ServerCore + ServeRegistry of this process (rs_cluster)."""

    def __init__(self, pipeline: bool = True, smart_skipping: bool = True):
        h = C.c_void_p()
        check(lib.rs_cluster_create(int(pipeline), int(smart_skipping), C.byref(h)))
        self.h = h
        self.handles: list[Handle] = []

    def close(self):
        for hd in list(self.handles):
            hd.close()
        if self.h:
            lib.rs_cluster_destroy(self.h)
            self.h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def open(self, model: str, replica: str, num_shards: int = 1, **cfg) -> "Handle":
        out = C.c_void_p()
        c = make_config(**cfg)
        check(lib.rs_open(self.h, _b(model), _b(replica), num_shards, C.byref(c), C.byref(out)),
              "rs_open")
        hd = Handle(self, out, model, replica, num_shards)
        self.handles.append(hd)
        return hd

    # ---- introspection -------------------------------------------------
    def trace(self) -> str:
        return _read_bytes(lib.rs_cluster_trace, self.h).decode()

    def assigns(self) -> list[Assign]:
        out = []
        for line in self.trace().splitlines():
            m = _ASSIGN.match(line)
            if m:
                kv = dict(f.split("=", 1) for f in m.group(1).split())
                out.append(Assign(kv["replica"], int(kv["v"]), kv["src"], int(kv["src_serving"])))
        return out

    def listing(self, model: str = "m") -> dict[int, set[str]]:
        text = _read_bytes(lib.rs_cluster_listing, self.h, _b(model)).decode()
        out: dict[int, set[str]] = {}
        for part in filter(None, text.split(";")):
            v, reps = part.split(":", 1)
            out[int(v)] = set(filter(None, reps.split(",")))
        return out

    def view(self, model: str, replica: str) -> Optional[dict]:
        life = C.create_string_buffer(16)
        v, s, vis = C.c_uint64(), C.c_uint32(), C.c_int()
        rc = lib.rs_cluster_view(self.h, _b(model), _b(replica), life, C.byref(v), C.byref(s),
                                 C.byref(vis))
        if rc == Status.not_found:
            return None
        check(rc)
        kind = _read_bytes(lib.rs_cluster_kind, self.h, _b(model), _b(replica)).decode()
        seeding = C.c_int()
        check(lib.rs_cluster_seeding(self.h, _b(model), _b(replica), C.byref(seeding)))
        return {"kind": kind, "lifecycle": life.value.decode(), "version": v.value,
                "serving": s.value, "visible": bool(vis.value), "seeding": bool(seeding.value)}

    def progress(self, model: str, replica: str) -> int:
        """The replica's verified items (min over shards), as its fills report."""
        v = C.c_uint64()
        check(lib.rs_cluster_progress(self.h, _b(model), _b(replica), C.byref(v)))
        return v.value

    def listen(self, host: str = "127.0.0.1", port: int = 0) -> int:
        """Serve this process's serve states over TCP; returns the port.
        Sources whose endpoint is "tcp:<host>:<port>" are pulled through it."""
        p = C.c_int()
        check(lib.rs_cluster_listen(self.h, _b(host), port, C.byref(p)), "rs_cluster_listen")
        return p.value

    def releases(self, model: str, owner: str) -> list[int]:
        """Retention offloads of `owner` the registry released (taken)."""
        n = C.c_size_t(0)
        buf = (C.c_uint64 * 64)()
        check(lib.rs_server_take_releases(self.h, _b(model), _b(owner), C.cast(buf, C.c_void_p), 64,
                                          C.byref(n)))
        return [int(buf[i]) for i in range(min(n.value, 64))]

    def locate(self, model: str, replica: str, spec: str = "latest", shard: int = 0) -> dict:
        a = RsAssignment()
        check(lib.rs_locate(self.h, _b(model), _b(replica), _b(spec), shard, C.byref(a)), "rs_locate")
        return _assignment(a)

    def set_topology(self, endpoints, cost) -> None:
        """The planner's source cost between data endpoints:
        cost[i][j] for a reader at endpoints[i] pulling from endpoints[j]
        (see nvlink_cost_matrix).  [] clears it."""
        n = len(endpoints)
        eps = (C.c_char_p * max(n, 1))(*[_b(e) for e in endpoints])
        flat = (C.c_int32 * max(n * n, 1))(*[int(cost[i][j]) for i in range(n) for j in range(n)])
        check(lib.rs_cluster_set_topology(self.h, n, C.cast(eps, C.c_void_p), C.cast(flat, C.c_void_p)),
              "rs_cluster_set_topology")

    def set_silent(self, model: str, replica: str, silent: bool = True):
        check(lib.rs_cluster_set_silent(self.h, _b(model), _b(replica), int(silent)))


def _assignment(a: RsAssignment) -> dict:
    return {"version": a.version, "source_replica": a.source_replica.decode(),
            "source_endpoint": a.source_endpoint.decode(), "source_complete": bool(a.source_complete),
            "cross_dc": bool(a.cross_dc), "seeding": bool(a.seeding),
            "local_seed_consume": bool(a.local_seed_consume)}


class Handle:
    """ClientCore for one replica (rs_handle).  Registered tensors are
    caller-owned CUDA memory that must outlive the handle."""

    def __init__(self, cluster: Cluster, h, model: str, replica: str, num_shards: int):
        self.cluster = cluster
        self.h = h
        self.model = model
        self.replica = replica
        self.num_shards = num_shards
        self._keep = []
        self.retain = []

    # ---- setup ------------------------------------------------------------
    def register_tensor(self, shard: int, name: str, tensor=None, *, ptr: int = 0,
                        nbytes: int = 0) -> Status:
        if tensor is not None:
            if not tensor.is_cuda or not tensor.is_contiguous():
                return Status.invalid_argument
            ptr, nbytes = tensor.data_ptr(), tensor.numel() * tensor.element_size()
            self._keep.append(tensor)
        return Status(lib.rs_register(self.h, shard, _b(name), C.c_void_p(ptr), nbytes))

    def register_slice(self, shard: int, name: str, tensor, geometry) -> Status:
        """Register a region holding a slice of a logical tensor;
        geometry = (rows, row_bytes, r0, nr, c0, nc) as from tp_slice()."""
        if not tensor.is_cuda or not tensor.is_contiguous():
            return Status.invalid_argument
        self._keep.append(tensor)
        rows, w, r0, nr, c0, nc = (int(x) for x in geometry)
        return Status(lib.rs_register_slice(self.h, shard, _b(name), C.c_void_p(tensor.data_ptr()),
                                            tensor.numel() * tensor.element_size(), rows, w, r0, nr,
                                            c0, nc))

    def register_cast(self, shard: int, name: str, tensor, nbytes: int, geometry=None) -> Status:
        """Register an fp8 e4m3 region (uint8 / float8_e4m3fn, nbytes/2
        bytes) that receives the version's bf16 entry `name` (nbytes bf16
        bytes) cast on landing (K5).  geometry as for register_slice, or None.
        The replica becomes terminal: it pulls, never serves or publishes."""
        if not tensor.is_cuda or not tensor.is_contiguous():
            return Status.invalid_argument
        if tensor.numel() * tensor.element_size() * 2 != nbytes:
            return Status.invalid_argument
        self._keep.append(tensor)
        rows, w, r0, nr, c0, nc = (int(x) for x in (geometry or (0, 0, 0, 0, 0, 0)))
        return Status(lib.rs_register_cast(self.h, shard, _b(name), C.c_void_p(tensor.data_ptr()),
                                           nbytes, rows, w, r0, nr, c0, nc))

    def set_retention(self, lags) -> None:
        """RetentionRule: keep the versions at these lags behind the newest
        published one reachable (call before the first op)."""
        arr = (C.c_uint64 * max(len(lags), 1))(*[int(x) for x in lags])
        check(lib.rs_set_retention(self.h, C.cast(arr, C.c_void_p), len(lags)))
        self.retain = sorted(int(x) for x in lags)

    def connect(self) -> Status:
        """ClientCore::open: join the cluster without an operation."""
        return Status(lib.rs_connect(self.h))

    def lanes(self) -> list[int]:
        """Versions this handle holds as retention offloads in host memory."""
        n = C.c_size_t(0)
        buf = (C.c_uint64 * 64)()
        check(lib.rs_lanes(self.h, C.cast(buf, C.c_void_p), 64, C.byref(n)))
        return [int(buf[i]) for i in range(min(n.value, 64))]

    def poll(self) -> None:
        """Free the retention offloads and seed buffers the registry released."""
        check(lib.rs_poll(self.h))

    def seed_lanes(self) -> list[int]:
        """Versions this handle holds as cross-link seed buffers in host
        memory (waits for a running seed fill first)."""
        n = C.c_size_t(0)
        buf = (C.c_uint64 * 64)()
        check(lib.rs_seed_lanes(self.h, C.cast(buf, C.c_void_p), 64, C.byref(n)))
        return [int(buf[i]) for i in range(min(n.value, 64))]

    def seed_wait(self) -> None:
        """Wait for a running seed fill (and its report to the registry)."""
        check(lib.rs_seed_wait(self.h))

    def local_shards(self) -> list[int]:
        """Shards whose regions this process registered (a replica may span
        several processes, one per GPU)."""
        return [s for s in range(self.num_shards) if lib.rs_shard_local(self.h, s)]

    def shard_hash(self, shard: int) -> tuple[int, bool, bool]:
        """(hash, has geometry, has cast) of one shard's registrations."""
        hv, g, c = C.c_uint64(), C.c_int(), C.c_int()
        check(lib.rs_shard_hash(self.h, shard, C.byref(hv), C.byref(g), C.byref(c)))
        return hv.value, bool(g.value), bool(c.value)

    def layout(self, shard: int = 0) -> bytes:
        return _read_bytes(lib.rs_layout, self.h, shard)

    def derived(self, shard: int, what: int) -> bytes:
        """Own-slicing derived manifest (0) / layout (1) of a shard."""
        return _read_bytes(lib.rs_derived, self.h, shard, what)

    @property
    def layout_key(self) -> str:
        return _read_bytes(lib.rs_layout_key, self.h).decode()

    def set_endpoint(self, shard: int, endpoint: str):
        check(lib.rs_set_endpoint(self.h, shard, _b(endpoint)))

    def set_stream(self, shard: int, stream) -> None:
        raw = stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
        check(lib.rs_set_stream(self.h, shard, C.c_void_p(raw)))

    # ---- ops --------------------------------------------------------------
    def publish(self, version: int) -> OpResult:
        st = Status(lib.rs_publish(self.h, version))
        return OpResult(st, version if st == Status.ok else None)

    def unpublish(self) -> OpResult:
        return OpResult(Status(lib.rs_unpublish(self.h)))

    @property
    def publish_pending(self) -> bool:
        """Early publish: the last publish still digests its big entries."""
        return bool(lib.rs_publish_pending(self.h))

    def set_early_publish(self, on: bool) -> None:
        """rs_config.early_publish for the next publish."""
        check(lib.rs_set_early_publish(self.h, int(on)))

    def finalize(self, wait_s: float = 60.0) -> Status:
        """Early publish: wait for the big-entry digests and commit the final
        (reference-identical) manifests."""
        return Status(lib.rs_publish_finalize(self.h, wait_s))

    def replicate(self, spec: str = "latest", wait_s: float = 60.0) -> OpResult:
        v = C.c_uint64()
        st = Status(lib.rs_replicate(self.h, _b(spec), wait_s, C.byref(v)))
        return OpResult(st, v.value if st == Status.ok else None)

    def update(self, spec: str = "latest", wait_s: float = 60.0) -> OpResult:
        v, ch = C.c_uint64(), C.c_int()
        st = Status(lib.rs_update(self.h, _b(spec), wait_s, C.byref(ch), C.byref(v)))
        return OpResult(st, v.value if st == Status.ok and v.value else None, bool(ch.value))

    def close(self) -> OpResult:
        if not self.h:
            return OpResult(Status.closed)
        st = Status(lib.rs_close(self.h))
        self.h = None
        if self in self.cluster.handles:
            self.cluster.handles.remove(self)
        return OpResult(st)

    def invalidate(self):
        check(lib.rs_invalidate(self.h))

    # ---- split phase (the caller drives the registry: rs_server_* / rs_transfer_*)
    def server_replicate(self, spec: str = "latest", update: bool = False) -> OpResult:
        """Plan this replica's replicate/update on the in-process registry
        without filling (ServerCore side of ClientCore::replicate)."""
        c, m, r = self.cluster.h, _b(self.model), _b(self.replica)
        if update:
            cur = self.current_version
            rc = lib.rs_server_update(c, m, r, _b(spec), int(cur is not None), cur or 0)
        else:
            rc = lib.rs_server_replicate(c, m, r, _b(spec))
        if rc:
            return OpResult(Status(rc))
        d, s, v, ch = C.c_int(), C.c_int(), C.c_uint64(), C.c_int()
        check(lib.rs_server_result(c, m, r, C.byref(d), C.byref(s), C.byref(v), C.byref(ch)))
        if not d.value:
            return OpResult(Status.timeout)
        return OpResult(Status(s.value), v.value if s.value == 0 else None, bool(ch.value))

    def transfer_bind(self, version: int) -> Status:
        """Bind every local shard to its assignment; the (empty) fill is
        served at once, so downstream readers can chase it."""
        return Status(lib.rs_transfer_bind(self.h, version))

    def transfer_launch(self) -> Status:
        """Launch the pending shards' pull kernels; returns while they run."""
        return Status(lib.rs_transfer_launch(self.h))

    def transfer_progress(self, shard: int = 0) -> tuple[int, int]:
        """(verified batches, batches) of the shard's running fill."""
        done, n = C.c_uint32(), C.c_uint32()
        check(lib.rs_transfer_progress(self.h, shard, C.byref(done), C.byref(n)))
        return done.value, n.value

    def transfer_wait(self) -> list[tuple[Status, int]]:
        """Wait for the launched fills: (status, reason) per shard."""
        n = self.num_shards
        sts, rsn = (C.c_int * n)(), (C.c_int * n)()
        lib.rs_transfer_wait(self.h, C.cast(sts, C.c_void_p), C.cast(rsn, C.c_void_p))
        return [(Status(sts[i]), int(rsn[i])) for i in range(n)]

    def transfer_assignment(self, shard: int = 0) -> dict:
        """The assignment the shard's latest fill was launched on."""
        a = RsAssignment()
        check(lib.rs_transfer_assignment(self.h, shard, C.byref(a)), "rs_transfer_assignment")
        return _assignment(a)

    def transfer_finish(self, version: int, good: bool) -> None:
        """Finish the fill (serve complete / stop serving) and report every
        shard's completion to the registry."""
        check(lib.rs_transfer_finish(self.h, version, int(good)))
        st = 0 if good else int(Status.transfer_failed)
        for s in range(self.num_shards):
            lib.rs_server_complete(self.cluster.h, _b(self.model), _b(self.replica), s, st)

    # ---- introspection ----------------------------------------------------
    @property
    def current_version(self) -> Optional[int]:
        v = C.c_uint64()
        return v.value if lib.rs_current_version(self.h, C.byref(v)) == 0 else None

    @property
    def is_published(self) -> bool:
        return bool(lib.rs_is_published(self.h))

    def stats(self) -> Stats:
        s = RsStats()
        check(lib.rs_stats_get(self.h, C.byref(s)))
        return Stats(**{f: getattr(s, f) for f, _ in RsStats._fields_})

    def manifest(self, shard: int = 0) -> bytes:
        return _read_bytes(lib.rs_manifest, self.h, shard)

    def chunk_digests(self, shard: int = 0):
        import numpy as np
        n = C.c_size_t(0)
        check(lib.rs_chunk_digests(self.h, shard, None, 0, C.byref(n)))
        out = np.zeros(n.value, np.uint64)
        check(lib.rs_chunk_digests(self.h, shard, out.ctypes.data, n.value, C.byref(n)))
        return out

    def serve_export(self, shard: int = 0) -> bytes:
        return _read_bytes(lib.rs_serve_export, self.h, shard)


def nvlink_cost_matrix(n: int = None) -> list[list[int]]:
    """The box's GPU-to-GPU topology measured through NVML: 0 for the same
    GPU (local HBM), 1 for a pair joined by NVLink (directly or through
    NVSwitch: every pair of a B200 HGX box), 2 for a pair that only reaches
    over PCIe.  The planner prefers lower costs (Cluster.set_topology)."""
    import pynvml as N
    N.nvmlInit()
    try:
        count = N.nvmlDeviceGetCount() if n is None else n
        hs = [N.nvmlDeviceGetHandleByIndex(i) for i in range(count)]
        out = [[0] * count for _ in range(count)]
        for i in range(count):
            for j in range(count):
                if i == j:
                    continue
                try:
                    st = N.nvmlDeviceGetP2PStatus(hs[i], hs[j], N.NVML_P2P_CAPS_INDEX_NVLINK)
                except N.NVMLError:
                    st = None
                out[i][j] = 1 if st == N.NVML_P2P_STATUS_OK else 2
        return out
    finally:
        N.nvmlShutdown()


def combine_layout_key(shard_hashes) -> str:
    """Slicing key of a replica from its shards' (hash, geometry, cast), in
    shard order (the key Handle.layout_key computes when one process holds
    every shard)."""
    n = len(shard_hashes)
    hs = (C.c_uint64 * max(n, 1))(*[int(h[0]) for h in shard_hashes])
    gs = (C.c_int * max(n, 1))(*[int(bool(h[1])) for h in shard_hashes])
    cs = (C.c_int * max(n, 1))(*[int(bool(h[2])) for h in shard_hashes])
    return _read_bytes(lib.rs_combine_layout_key, n, C.cast(hs, C.c_void_p), C.cast(gs, C.c_void_p),
                       C.cast(cs, C.c_void_p)).decode()


# ----------------------------------------------------------------------------
# Device primitives
def digest_spans(ptrs, lens, device: int = 0) -> list[int]:
    import numpy as np
    p = np.asarray(ptrs, np.uint64)
    n = np.asarray(lens, np.uint64)
    out = np.zeros(len(p), np.uint64)
    check(lib.rs_digest_spans(p.ctypes.data, n.ctypes.data, len(p), out.ctypes.data, device),
          "rs_digest_spans")
    return [int(x) for x in out]


def synth_bf16(tensor, seed: int, first: int = 0, stream=None):
    """Fill a contiguous CUDA tensor (any dtype; viewed as bf16 words) with
    the synthetic weights of SURVEY.md §8d."""
    n = tensor.numel() * tensor.element_size() // 2
    raw = 0 if stream is None else stream.cuda_stream
    check(lib.rs_synth_bf16(C.c_void_p(tensor.data_ptr()), n, seed, first, C.c_void_p(raw)),
          "rs_synth_bf16")


def bf16_to_e4m3(src, dst, stream=None):
    """K5 standalone: dst (n bytes) = e4m3 of the n bf16 words of src (a
    contiguous CUDA tensor of any dtype, viewed as bf16 words)."""
    n = src.numel() * src.element_size() // 2
    if dst.numel() * dst.element_size() < n:
        raise ValueError("dst holds fewer bytes than src has bf16 words")
    raw = 0 if stream is None else stream.cuda_stream
    check(lib.rs_bf16_to_e4m3(C.c_void_p(src.data_ptr()), C.c_void_p(dst.data_ptr()), n,
                              C.c_void_p(raw)), "rs_bf16_to_e4m3")


def pull_spans(srcs, dsts, lens, chunk_bytes=4096, expect=None, out_digests=None, device=0,
               stream=None):
    """Standalone fused copy+verify over explicit device spans.  Returns
    (kernel_code, kernel_ms)."""
    import numpy as np
    import torch
    s = np.asarray(srcs, np.uint64)
    d = np.asarray(dsts, np.uint64) if dsts is not None else None
    n = np.asarray(lens, np.uint64)
    # dense (caller) <-> batch-aligned (kernel) chunk-table index maps
    idx, base = [], 0
    for ln in lens:
        cnt = (int(ln) + chunk_bytes - 1) // chunk_bytes
        idx.extend(range(base, base + cnt))
        base += (cnt + 31) // 32 * 32
    dev = torch.device("cuda", device)
    pos = torch.tensor(idx, dtype=torch.int64, device=dev)
    exp_al = out_al = None
    if expect is not None:
        exp_al = torch.zeros(max(base, 1), dtype=torch.int64, device=dev)
        exp_al[pos] = expect
    if out_digests is not None:
        out_al = torch.zeros(max(base, 1), dtype=torch.int64, device=dev)
    torch.cuda.synchronize(dev)
    code, ms = C.c_int(), C.c_float()
    raw = 0 if stream is None else stream.cuda_stream
    check(lib.rs_pull_spans(s.ctypes.data, None if d is None else d.ctypes.data, n.ctypes.data,
                            len(s), chunk_bytes,
                            None if exp_al is None else C.c_void_p(exp_al.data_ptr()),
                            None if out_al is None else C.c_void_p(out_al.data_ptr()),
                            device, C.c_void_p(raw), C.byref(code), C.byref(ms)), "rs_pull_spans")
    if out_al is not None:
        out_digests.copy_(out_al[pos])
    return code.value, ms.value
