"""TEST INFRASTRUCTURE ONLY -- ctypes access to the CPU oracle.

Two libraries, both built by ``make -C oracle`` (``__graft_entry__.build()``):

* ``_port/libros_oracle.so`` -- our plain-C restatement (ros_oracle.c).
* ``_ref/librefstore_ref.so`` -- the UNMODIFIED reference refstore sources
  compiled from /root/reference/proj/src, plus ``ref_shim.cpp``'s C ABI.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (cpu_baseline /
``--impl reference``) may import this module, and only as the checker or the
CPU baseline -- never as the thing measured or shipped.
"""
from __future__ import annotations

import ctypes as C
import os
import re
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "_port", "libros_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "librefstore_ref.so")

u8p = C.POINTER(C.c_uint8)
u16p = C.POINTER(C.c_uint16)
u64p = C.POINTER(C.c_uint64)

_port = None
_ref = None


def _ptr(a: np.ndarray, t=C.c_void_p):
    return C.cast(a.ctypes.data, t)


def port():
    global _port
    if _port is None:
        lib = C.CDLL(PORT_SO)
        lib.ro_xxh64.restype = C.c_uint64
        lib.ro_xxh64.argtypes = [C.c_void_p, C.c_size_t]
        lib.ro_splitmix_bytes.argtypes = [C.c_uint64, C.c_size_t, C.c_void_p]
        lib.ro_pattern_bytes.argtypes = [C.c_size_t, C.c_void_p]
        lib.ro_fill_pattern.argtypes = [C.c_uint64, C.c_size_t, C.c_void_p]
        lib.ro_synth_bf16.argtypes = [C.c_uint64, C.c_uint64, C.c_size_t, C.c_void_p]
        lib.ro_chunk_digests.restype = C.c_size_t
        lib.ro_chunk_digests.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_uint64, C.c_void_p]
        lib.ro_assemble.restype = C.c_int
        lib.ro_assemble.argtypes = [C.c_size_t, C.c_void_p, C.c_uint64, C.c_uint64, C.c_void_p, C.c_void_p]
        lib.ro_manifest_encode.restype = C.c_size_t
        lib.ro_manifest_encode.argtypes = [C.c_size_t, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                           C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]
        lib.ro_bf16_to_e4m3.argtypes = [C.c_void_p, C.c_size_t, C.c_void_p]
        lib.ro_chunk_len_for.restype = C.c_uint32
        lib.ro_chunk_len_for.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint32]
        _port = lib
    return _port


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref():
    global _ref
    if _ref is None:
        lib = C.CDLL(REF_SO)
        lib.ref_digest64.restype = C.c_uint64
        lib.ref_digest64.argtypes = [C.c_void_p, C.c_size_t]
        lib.ref_build_manifest.restype = C.c_long
        lib.ref_build_manifest.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64,
                                           C.c_uint64, C.c_char_p, C.c_size_t]
        lib.ref_build_manifest_pre.restype = C.c_long
        lib.ref_build_manifest_pre.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                               C.c_uint64, C.c_uint64, C.c_char_p, C.c_size_t]
        lib.ref_assemble_manifest.restype = C.c_long
        lib.ref_assemble_manifest.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64,
                                              C.c_uint64, C.c_int, C.c_char_p, C.c_size_t]
        lib.ref_modeled_entry_digest.restype = C.c_uint64
        lib.ref_modeled_entry_digest.argtypes = [C.c_char_p, C.c_uint64, C.c_uint64]
        lib.ref_manifest_items.restype = C.c_long
        lib.ref_manifest_items.argtypes = [C.c_char_p, C.c_size_t, C.c_void_p, C.c_size_t]
        lib.ref_version_resolve.restype = C.c_int
        lib.ref_version_resolve.argtypes = [C.c_char_p, C.c_void_p, C.c_int, C.c_void_p]
        lib.ref_cluster_new.restype = C.c_void_p
        lib.ref_cluster_new.argtypes = [C.c_int, C.c_int, C.c_int, C.c_uint64]
        lib.ref_cluster_add.argtypes = [C.c_void_p, C.c_char_p, C.c_uint32, C.c_uint64, C.c_uint64]
        lib.ref_cluster_add_dc.argtypes = [C.c_void_p, C.c_char_p, C.c_uint32, C.c_char_p, C.c_int]
        lib.ref_cluster_register.argtypes = [C.c_void_p, C.c_char_p, C.c_uint32, C.c_char_p, C.c_void_p,
                                             C.c_uint64]
        lib.ref_cluster_register_modeled.argtypes = [C.c_void_p, C.c_char_p, C.c_uint32, C.c_char_p,
                                                     C.c_uint64]
        lib.ref_cluster_publish.argtypes = [C.c_void_p, C.c_char_p, C.c_uint64, C.c_void_p]
        lib.ref_cluster_unpublish.argtypes = [C.c_void_p, C.c_char_p]
        lib.ref_cluster_close.argtypes = [C.c_void_p, C.c_char_p]
        lib.ref_cluster_set_retention.argtypes = [C.c_void_p, C.c_char_p, C.c_void_p, C.c_int]
        lib.ref_cluster_open.argtypes = [C.c_void_p, C.c_char_p]
        lib.ref_cluster_pull_many.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_char_p, C.c_int,
                                              C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        lib.ref_cluster_settle.argtypes = [C.c_void_p]
        lib.ref_cluster_trace.restype = C.c_long
        lib.ref_cluster_trace.argtypes = [C.c_void_p, C.c_char_p, C.c_size_t]
        lib.ref_cluster_stats.argtypes = [C.c_void_p, C.c_char_p, C.c_void_p]
        lib.ref_cluster_view.restype = C.c_long
        lib.ref_cluster_view.argtypes = [C.c_void_p, C.c_char_p, C.c_void_p, C.c_void_p, C.c_char_p,
                                         C.c_size_t]
        lib.ref_cluster_free.argtypes = [C.c_void_p]
        _ref = lib
    return _ref


# ------------------------------------------------------------------ port API
def xxh64(data) -> int:
    b = np.ascontiguousarray(np.frombuffer(bytes(data), np.uint8) if isinstance(data, (bytes, bytearray))
                             else data).view(np.uint8)
    return int(port().ro_xxh64(b.ctypes.data, b.nbytes))


def splitmix_bytes(seed: int, n: int) -> bytes:
    out = np.empty(n, np.uint8)
    port().ro_splitmix_bytes(seed, n, out.ctypes.data)
    return out.tobytes()


def pattern_bytes(n: int) -> bytes:
    out = np.empty(n, np.uint8)
    port().ro_pattern_bytes(n, out.ctypes.data)
    return out.tobytes()


def fill_pattern(salt: int, n: int) -> np.ndarray:
    out = np.empty(n, np.uint8)
    port().ro_fill_pattern(salt, n, out.ctypes.data)
    return out


def synth_bf16(seed: int, n: int, first: int = 0) -> np.ndarray:
    out = np.empty(n, np.uint16)
    port().ro_synth_bf16(seed, first, n, out.ctypes.data)
    return out


def chunk_digests(items: list[np.ndarray], chunk: int) -> np.ndarray:
    arrs = [np.ascontiguousarray(a).view(np.uint8).reshape(-1) for a in items]
    ptrs = np.array([a.ctypes.data for a in arrs], np.uint64)
    lens = np.array([a.nbytes for a in arrs], np.uint64)
    n = port().ro_chunk_digests(ptrs.ctypes.data, lens.ctypes.data, len(arrs), chunk, None)
    out = np.empty(n, np.uint64)
    port().ro_chunk_digests(ptrs.ctypes.data, lens.ctypes.data, len(arrs), chunk, out.ctypes.data)
    return out


def assemble(lens, tiny=2 << 20, target=64 << 20):
    lens = np.asarray(lens, np.uint64)
    g = np.empty(len(lens), np.int32)
    off = np.empty(len(lens), np.uint64)
    ng = port().ro_assemble(len(lens), lens.ctypes.data, tiny, target, g.ctypes.data, off.ctypes.data)
    return ng, g, off


def manifest_encode(names, lens, digests, group_of, offset, n_groups, group_digests) -> bytes:
    cnames = (C.c_char_p * len(names))(*[n.encode() for n in names])
    lens = np.asarray(lens, np.uint64)
    digests = np.asarray(digests, np.uint64)
    group_of = np.asarray(group_of, np.int32)
    offset = np.asarray(offset, np.uint64)
    gd = np.asarray(group_digests, np.uint64) if n_groups else np.zeros(1, np.uint64)
    args = (len(names), C.cast(cnames, C.c_void_p), lens.ctypes.data, digests.ctypes.data,
            group_of.ctypes.data, offset.ctypes.data, n_groups, gd.ctypes.data)
    n = port().ro_manifest_encode(*args, None)
    out = np.empty(n, np.uint8)
    port().ro_manifest_encode(*args, out.ctypes.data)
    return out.tobytes()


def publish_manifest(names, arrays, tiny=2 << 20, target=64 << 20) -> bytes:
    """build_publish_payload (client_core.cpp:1547-1579) restated with the port."""
    arrs = [np.ascontiguousarray(a).view(np.uint8).reshape(-1) for a in arrays]
    lens = [a.nbytes for a in arrs]
    digests = [xxh64(a) for a in arrs]
    ng, g, off = assemble(lens, tiny, target)
    gds = []
    for k in range(ng):
        staging = np.concatenate([arrs[e] for e in range(len(arrs)) if g[e] == k])
        gds.append(xxh64(staging))
    return manifest_encode(names, lens, digests, g, off, ng, gds)


def chunk_len_for(row_bytes: int, nc: int, chunk_bytes: int = 4096, align: int = 2) -> int:
    """The reshard chunk rule (ros_oracle.h ro_chunk_len_for)."""
    return int(port().ro_chunk_len_for(row_bytes, nc, chunk_bytes, align))


def slice_bytes(full: np.ndarray, geometry) -> np.ndarray:
    """Bytes a region with geometry (rows, row_bytes, r0, nr, c0, nc) holds,
    cut from the logical tensor's bytes `full` (row-major)."""
    rows, w, r0, nr, c0, nc = geometry
    b = np.ascontiguousarray(full).view(np.uint8).reshape(rows, w)
    return np.ascontiguousarray(b[r0:r0 + nr, c0:c0 + nc]).reshape(-1)


def chunk_digests_lens(items: list[np.ndarray], lens: list[int]) -> np.ndarray:
    """Chunk digests with a chunk length per item (concatenated, item order)."""
    out = [chunk_digests([a], int(l)) for a, l in zip(items, lens)]
    return np.concatenate(out) if out else np.zeros(0, np.uint64)


def bf16_to_e4m3(x: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(x, np.uint16)
    out = np.empty(x.shape, np.uint8)
    port().ro_bf16_to_e4m3(x.ctypes.data, x.size, out.ctypes.data)
    return out


# ------------------------------------------------------------- reference API
def ref_digest64(data) -> int:
    b = np.ascontiguousarray(np.frombuffer(bytes(data), np.uint8) if isinstance(data, (bytes, bytearray))
                             else data).view(np.uint8)
    return int(ref().ref_digest64(b.ctypes.data, b.nbytes))


def ref_build_manifest(names, arrays, tiny=2 << 20, target=64 << 20) -> bytes:
    arrs = [np.ascontiguousarray(a).view(np.uint8).reshape(-1) for a in arrays]
    cnames = (C.c_char_p * len(names))(*[n.encode() for n in names])
    ptrs = np.array([a.ctypes.data for a in arrs], np.uint64)
    lens = np.array([a.nbytes for a in arrs], np.uint64)
    args = (len(names), C.cast(cnames, C.c_void_p), ptrs.ctypes.data, lens.ctypes.data, tiny, target)
    n = ref().ref_build_manifest(*args, None, 0)
    assert n >= 0, n
    buf = C.create_string_buffer(n)
    ref().ref_build_manifest(*args, buf, n)
    return buf.raw[:n]


def ref_build_manifest_pre(names, lens, digests, tiny_arrays: dict, tiny=2 << 20,
                           target=64 << 20) -> bytes:
    """build_publish_payload with precomputed (reference digest64) entry
    digests; tiny_arrays maps entry index -> bytes for the group members."""
    keep = {i: np.ascontiguousarray(a).view(np.uint8).reshape(-1) for i, a in tiny_arrays.items()}
    cnames = (C.c_char_p * len(names))(*[n.encode() for n in names])
    ptrs = np.array([keep[i].ctypes.data if i in keep else 0 for i in range(len(names))], np.uint64)
    lens = np.asarray(lens, np.uint64)
    digests = np.asarray(digests, np.uint64)
    args = (len(names), C.cast(cnames, C.c_void_p), ptrs.ctypes.data, lens.ctypes.data,
            digests.ctypes.data, tiny, target)
    n = ref().ref_build_manifest_pre(*args, None, 0)
    assert n >= 0, n
    buf = C.create_string_buffer(n)
    ref().ref_build_manifest_pre(*args, buf, n)
    return buf.raw[:n]


def ref_assemble_manifest(names, lens, digests, tiny=2 << 20, target=64 << 20, seal=False) -> bytes:
    cnames = (C.c_char_p * len(names))(*[n.encode() for n in names])
    lens = np.asarray(lens, np.uint64)
    digests = np.asarray(digests, np.uint64)
    args = (len(names), C.cast(cnames, C.c_void_p), lens.ctypes.data, digests.ctypes.data, tiny, target,
            int(seal))
    n = ref().ref_assemble_manifest(*args, None, 0)
    assert n >= 0, n
    buf = C.create_string_buffer(n)
    ref().ref_assemble_manifest(*args, buf, n)
    return buf.raw[:n]


def ref_manifest_items(data: bytes) -> np.ndarray:
    n = ref().ref_manifest_items(data, len(data), None, 0)
    assert n >= 0, n
    out = np.empty((n, 5), np.uint64)
    ref().ref_manifest_items(data, len(data), out.ctypes.data, n)
    return out


_ASSIGN_RE = re.compile(r"^\d+ \d+ (\S+) assign (.*)$")


@dataclass
class Assign:
    replica: str
    version: int
    src: str
    src_serving: int


class RefCluster:
    """The reference ClusterFix (test_client_core.cpp:23-117) as an object."""

    def __init__(self, threaded=False, server_pipeline=True, client_pipeline=True, chunk_bytes=0):
        self.lib = ref()
        self.h = self.lib.ref_cluster_new(int(threaded), int(server_pipeline), int(client_pipeline),
                                          chunk_bytes)
        self._keep = []

    def close(self):
        if self.h:
            self.lib.ref_cluster_free(self.h)
            self.h = None

    def __del__(self):
        self.close()

    def add(self, replica, shards=1, tiny=0, target=0):
        self.lib.ref_cluster_add(self.h, replica.encode(), shards, tiny, target)

    def add_dc(self, replica, shards=1, dc="dc0", offload_seed=False):
        """A replica with ClientConfig.datacenter / offload_seed set."""
        self.lib.ref_cluster_add_dc(self.h, replica.encode(), shards, dc.encode(), int(offload_seed))

    def register(self, replica, shard, name, arr: np.ndarray):
        assert arr.flags.c_contiguous
        self._keep.append(arr)
        return self.lib.ref_cluster_register(self.h, replica.encode(), shard, name.encode(),
                                             arr.ctypes.data, arr.nbytes)

    def register_modeled(self, replica, shard, name, length):
        return self.lib.ref_cluster_register_modeled(self.h, replica.encode(), shard, name.encode(), length)

    def publish(self, replica, version):
        secs = C.c_double(0)
        st = self.lib.ref_cluster_publish(self.h, replica.encode(), version, C.byref(secs))
        return st, secs.value

    def unpublish(self, replica):
        return self.lib.ref_cluster_unpublish(self.h, replica.encode())

    def open(self, replica):
        return self.lib.ref_cluster_open(self.h, replica.encode())

    def close_replica(self, replica):
        """ClientCore::close: the replica leaves and stops serving."""
        return self.lib.ref_cluster_close(self.h, replica.encode())

    def set_retention(self, replica, lags):
        arr = (C.c_uint64 * max(len(lags), 1))(*lags)
        return self.lib.ref_cluster_set_retention(self.h, replica.encode(), C.cast(arr, C.c_void_p),
                                                  len(lags))

    def pull_many(self, replicas, spec="latest", update=False):
        n = len(replicas)
        names = (C.c_char_p * n)(*[r.encode() for r in replicas])
        st = np.zeros(n, np.int32)
        vs = np.zeros(n, np.uint64)
        ch = np.zeros(n, np.int32)
        secs = C.c_double(0)
        rc = self.lib.ref_cluster_pull_many(self.h, n, C.cast(names, C.c_void_p), spec.encode(), int(update),
                                            st.ctypes.data, vs.ctypes.data, ch.ctypes.data, C.byref(secs))
        assert rc == 0, rc
        return [int(x) for x in st], [int(x) for x in vs], [int(x) for x in ch], secs.value

    def settle(self):
        self.lib.ref_cluster_settle(self.h)

    def trace(self) -> str:
        n = self.lib.ref_cluster_trace(self.h, None, 0)
        buf = C.create_string_buffer(n + 1)
        self.lib.ref_cluster_trace(self.h, buf, n)
        return buf.raw[:n].decode()

    def assigns(self) -> list[Assign]:
        out = []
        for line in self.trace().splitlines():
            m = _ASSIGN_RE.match(line)
            if not m:
                continue
            kv = dict(f.split("=", 1) for f in m.group(2).split())
            out.append(Assign(kv["replica"], int(kv["v"]), kv["src"], int(kv["src_serving"])))
        return out

    def stats(self, replica) -> dict:
        out = np.zeros(7, np.uint64)
        self.lib.ref_cluster_stats(self.h, replica.encode(), out.ctypes.data)
        keys = ["bytes_pulled", "bytes_pulled_cross_dc", "bytes_copied_local", "items_verified",
                "checksum_failures", "failure_reports", "failovers"]
        return {k: int(v) for k, v in zip(keys, out)}

    def view(self, replica):
        v = C.c_uint64(0)
        s = C.c_uint32(0)
        buf = C.create_string_buffer(64)
        n = self.lib.ref_cluster_view(self.h, replica.encode(), C.byref(v), C.byref(s), buf, 64)
        if n < 0:
            return None
        return {"lifecycle": buf.raw[:n].decode(), "version": int(v.value), "serving": int(s.value)}
