"""ctypes binding of libros_b200.so (include/ros_b200.h).

There is no fallback: if the shared library is missing this import fails
loudly; build it with ``python -m paper_2604_09107_b200.build`` (or
``__graft_entry__.build()``).
"""
from __future__ import annotations

import ctypes as C
import os

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib", "libros_b200.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_2604_09107_b200.build` "
                      "(the B200 ROS path has no CPU fallback)")

lib = C.CDLL(LIB_PATH)

vp = C.c_void_p
u32, u64, i32, sz, dbl = C.c_uint32, C.c_uint64, C.c_int, C.c_size_t, C.c_double
cstr = C.c_char_p


class RsConfig(C.Structure):
    _fields_ = [("chunk_bytes", u64), ("tiny_threshold", u64), ("group_target", u64),
                ("pipeline", i32), ("checksum_retries", i32), ("pull_timeout_s", dbl),
                ("datacenter", C.c_char * 32), ("reshard_align", u32),
                ("grid_sms", u32), ("early_publish", i32), ("offload_seed", i32)]


class RsAssignment(C.Structure):
    _fields_ = [("version", u64), ("source_replica", C.c_char * 128),
                ("source_endpoint", C.c_char * 128), ("source_complete", i32), ("cross_dc", i32),
                ("seeding", i32), ("local_seed_consume", i32)]


class RsStats(C.Structure):
    _fields_ = [("bytes_pulled", u64), ("bytes_pulled_cross_dc", u64), ("bytes_copied_local", u64),
                ("items_verified", u64), ("checksum_failures", u64), ("failure_reports", u64),
                ("failovers", u64), ("last_pull_ms", C.c_float), ("last_publish_ms", C.c_float),
                ("last_pull_bytes", u64), ("last_pull_launches", u32), ("h2d_bytes", u64),
                ("d2h_bytes", u64), ("fill_max_ms", C.c_float), ("fill_sum_ms", C.c_float),
                ("fill_bytes", u64), ("kernel_launches", u64)]


_SIGS = {
    "rs_abi_version": (i32, []),
    "rs_status_name": (cstr, [i32]),
    "rs_config_default": (None, [C.POINTER(RsConfig)]),
    "rs_cluster_create": (i32, [i32, i32, C.POINTER(vp)]),
    "rs_cluster_destroy": (None, [vp]),
    "rs_cluster_trace": (i32, [vp, vp, sz, C.POINTER(sz)]),
    "rs_cluster_listing": (i32, [vp, cstr, vp, sz, C.POINTER(sz)]),
    "rs_cluster_view": (i32, [vp, cstr, cstr, vp, C.POINTER(u64), C.POINTER(u32), C.POINTER(i32)]),
    "rs_cluster_set_silent": (i32, [vp, cstr, cstr, i32]),
    "rs_cluster_set_topology": (i32, [vp, u32, vp, vp]),
    "rs_cluster_progress": (i32, [vp, cstr, cstr, C.POINTER(u64)]),
    "rs_cluster_seeding": (i32, [vp, cstr, cstr, C.POINTER(i32)]),
    "rs_cluster_source": (i32, [vp, cstr, cstr, vp, sz, C.POINTER(sz)]),
    "rs_open": (i32, [vp, cstr, cstr, u32, C.POINTER(RsConfig), C.POINTER(vp)]),
    "rs_register": (i32, [vp, u32, cstr, vp, u64]),
    "rs_register_slice": (i32, [vp, u32, cstr, vp, u64, u64, u64, u64, u64, u64, u64]),
    "rs_register_cast": (i32, [vp, u32, cstr, vp, u64, u64, u64, u64, u64, u64, u64]),
    "rs_layout_key": (i32, [vp, vp, sz, C.POINTER(sz)]),
    "rs_shard_local": (i32, [vp, u32]),
    "rs_set_retention": (i32, [vp, vp, sz]),
    "rs_connect": (i32, [vp]),
    "rs_pull": (i32, [vp, cstr, dbl, C.POINTER(u64)]),
    "rs_release": (i32, [vp, u64]),
    "rs_serve_state": (i32, [vp, u32, C.POINTER(vp), C.POINTER(vp), C.POINTER(u32), C.POINTER(u32)]),
    "rs_offload_lanes": (i32, [vp, u64]),
    "rs_lane_export": (i32, [vp, u32, u64, vp, sz, C.POINTER(sz)]),
    "rs_offload_release": (i32, [vp, u64]),
    "rs_poll": (i32, [vp]),
    "rs_lanes": (i32, [vp, vp, sz, C.POINTER(sz)]),
    "rs_seed_lanes": (i32, [vp, vp, sz, C.POINTER(sz)]),
    "rs_seed_wait": (i32, [vp]),
    "rs_seed_fill": (i32, [vp]),
    "rs_seed_status": (i32, [vp, u32]),
    "rs_seed_export": (i32, [vp, u32, u64, vp, sz, C.POINTER(sz)]),
    "rs_server_set_offload_seed": (i32, [vp, cstr, cstr, i32]),
    "rs_server_assignment": (i32, [vp, cstr, cstr, u32, C.POINTER(RsAssignment)]),
    "rs_server_seed_start": (i32, [vp, cstr, cstr, u32, C.POINTER(RsAssignment)]),
    "rs_server_seed_progress": (i32, [vp, cstr, cstr, u32, u64, u64]),
    "rs_server_seed_complete": (i32, [vp, cstr, cstr, u32, i32, u64]),
    "rs_server_set_retention": (i32, [vp, cstr, cstr, vp, sz]),
    "rs_server_offload_pending": (i32, [vp, cstr, cstr, C.POINTER(u64)]),
    "rs_server_offload_confirm": (i32, [vp, cstr, cstr, u32, u64, i32, cstr]),
    "rs_server_take_releases": (i32, [vp, cstr, cstr, vp, sz, C.POINTER(sz)]),
    "rs_cluster_kind": (i32, [vp, cstr, cstr, vp, sz, C.POINTER(sz)]),
    "rs_cluster_listen": (i32, [vp, cstr, i32, C.POINTER(i32)]),
    "rs_transfer_launch": (i32, [vp]),
    "rs_transfer_progress": (i32, [vp, u32, C.POINTER(u32), C.POINTER(u32)]),
    "rs_transfer_wait": (i32, [vp, vp, vp]),
    "rs_transfer_assignment": (i32, [vp, u32, C.POINTER(RsAssignment)]),
    "rs_shard_hash": (i32, [vp, u32, C.POINTER(u64), C.POINTER(i32), C.POINTER(i32)]),
    "rs_combine_layout_key": (i32, [u32, vp, vp, vp, vp, sz, C.POINTER(sz)]),
    "rs_chunk_len_for": (u32, [u64, u64, u64, u32]),
    "rs_layout": (i32, [vp, u32, vp, sz, C.POINTER(sz)]),
    "rs_transfer_derived": (i32, [vp]),
    "rs_set_endpoint": (i32, [vp, u32, cstr]),
    "rs_set_stream": (i32, [vp, u32, vp]),
    "rs_publish": (i32, [vp, u64]),
    "rs_unpublish": (i32, [vp]),
    "rs_replicate": (i32, [vp, cstr, dbl, C.POINTER(u64)]),
    "rs_update": (i32, [vp, cstr, dbl, C.POINTER(i32), C.POINTER(u64)]),
    "rs_close": (i32, [vp]),
    "rs_locate": (i32, [vp, cstr, cstr, cstr, u32, C.POINTER(RsAssignment)]),
    "rs_current_version": (i32, [vp, C.POINTER(u64)]),
    "rs_is_published": (i32, [vp]),
    "rs_stats_get": (i32, [vp, C.POINTER(RsStats)]),
    "rs_manifest": (i32, [vp, u32, vp, sz, C.POINTER(sz)]),
    "rs_manifest_now": (i32, [vp, u32, vp, sz, C.POINTER(sz)]),
    "rs_chunk_digests": (i32, [vp, u32, vp, sz, C.POINTER(sz)]),
    "rs_invalidate": (i32, [vp]),
    "rs_server_open": (i32, [vp, cstr, cstr, u32, cstr, vp, cstr, vp, vp, vp, vp]),
    "rs_derived": (i32, [vp, u32, i32, vp, sz, C.POINTER(sz)]),
    "rs_server_publish": (i32, [vp, cstr, cstr, u64, u32, vp, vp, vp, vp]),
    "rs_server_add_layout": (i32, [vp, cstr, u64, cstr, u32, vp, vp, vp, vp]),
    "rs_server_unpublish": (i32, [vp, cstr, cstr]),
    "rs_server_publish_provisional": (i32, [vp, cstr, cstr, u64, u32, vp, vp, vp, vp]),
    "rs_server_finalize": (i32, [vp, cstr, cstr, u64, u32, vp, vp]),
    "rs_publish_pending": (i32, [vp]),
    "rs_set_early_publish": (i32, [vp, i32]),
    "rs_publish_finalize": (i32, [vp, dbl]),
    "rs_server_replicate": (i32, [vp, cstr, cstr, cstr]),
    "rs_server_update": (i32, [vp, cstr, cstr, cstr, i32, u64]),
    "rs_server_result": (i32, [vp, cstr, cstr, C.POINTER(i32), C.POINTER(i32), C.POINTER(u64),
                               C.POINTER(i32)]),
    "rs_server_complete": (i32, [vp, cstr, cstr, u32, i32]),
    "rs_server_failure_report": (i32, [vp, cstr, cstr, u32, cstr, i32]),
    "rs_server_close": (i32, [vp, cstr, cstr]),
    "rs_prepare_publish": (i32, [vp, u64]),
    "rs_commit_publish": (i32, [vp, u64, i32]),
    "rs_transfer_bind": (i32, [vp, u64]),
    "rs_transfer_fill": (i32, [vp, vp, vp]),
    "rs_transfer_finish": (i32, [vp, u64, i32]),
    "rs_serve_export": (i32, [vp, u32, vp, sz, C.POINTER(sz)]),
    "rs_serve_import": (i32, [vp, vp, sz]),
    "rs_oplog_serve": (i32, [cstr, i32, C.POINTER(i32), C.POINTER(vp)]),
    "rs_oplog_server_stop": (None, [vp]),
    "rs_oplog_server_size": (u64, [vp]),
    "rs_oplog_connect": (i32, [cstr, i32, dbl, C.POINTER(vp)]),
    "rs_oplog_append": (i32, [vp, vp, sz, C.POINTER(u64)]),
    "rs_oplog_fetch": (i32, [vp, u64, i32, u32, C.POINTER(u64)]),
    "rs_oplog_entry": (i32, [vp, u64, C.POINTER(vp), C.POINTER(sz)]),
    "rs_oplog_close": (None, [vp]),
    "rs_digest_spans": (i32, [vp, vp, i32, vp, i32]),
    "rs_synth_bf16": (i32, [vp, u64, u64, u64, vp]),
    "rs_bf16_to_e4m3": (i32, [vp, vp, u64, vp]),
    "rs_pull_spans": (i32, [vp, vp, vp, i32, u64, vp, vp, i32, vp, C.POINTER(i32),
                            C.POINTER(C.c_float)]),
}

for _name, (_res, _args) in _SIGS.items():
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args

EXPORTED = tuple(_SIGS)
