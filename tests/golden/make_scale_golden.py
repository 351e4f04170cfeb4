"""Generates tests/golden/scale.json: parity fixtures at BASELINE config scale.

    python tests/golden/make_scale_golden.py      (needs oracle/_ref; ~5 min, 8 cores)

The bytes are the bench's synthetic workloads (SURVEY.md §8d generator, seed
42 + tensor index, made by the oracle's C restatement ro_synth_bf16, which the
GPU generator matches bit for bit):

* config 2 -- Llama-3-8B bf16, 291 tensors, 16,060,522,496 B, one replica;
* config 5 -- the Llama-3-70B TP-8 shard the bench publishes (17.64 GB bf16),
  landed as fp8 e4m3;
* config 3 -- Qwen2.5-32B bf16 (65.5 GB): the trainer's FSDP-8 shards
  (Shard(0) row blocks) and the TP-2 reader shards cut from the same tensors.

Every digest and manifest below is computed by the UNMODIFIED reference
(oracle/_ref): digest64 (digest.cpp:79-106), assemble_manifest + pack_group +
encode (manifest.cpp:103-215) -- i.e. build_publish_payload
(client_core.cpp:1547-1579) -- over those bytes.  What the reference has no
counterpart for is restated by the oracle (oracle/ros_oracle.c): the chunk
partition of the digest table (4096-byte item-relative chunks), the TP/FSDP
slice geometry and the bf16 -> e4m3 cast.  The GPU tests
(tests/test_scale_parity.py) compare the device-built manifests, chunk tables
and landed bytes against these values on the GPU box, where /root/reference
does not exist.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time
from multiprocessing import Pool

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402

import bench as B  # noqa: E402  (workload_shapes / tp_dim / tp_slice: the bench's own layouts)

CHUNK = 4096
TINY = 2 << 20


def _numel(shape):
    n = 1
    for d in shape:
        n *= d
    return n


def _tensor(job):
    """One tensor: generate, then reference digests of what the job asks for."""
    seed, shape = job["seed"], job["shape"]
    a = O.synth_bf16(seed, _numel(shape))
    out = {"i": job["i"], "digest": O.ref_digest64(a)}
    if job.get("chunks"):
        out["chunks"] = O.chunk_digests([a], CHUNK)
    if job.get("cast"):
        out["cast_digest"] = O.ref_digest64(O.bf16_to_e4m3(a))
    if a.nbytes < TINY:
        out["bytes"] = a
    for key, geo in job.get("slices", {}).items():
        s = O.slice_bytes(a, geo)
        out[key] = O.ref_digest64(s)
        if s.nbytes < TINY:
            out[key + "_bytes"] = s
    return out


def _run(jobs, pool):
    res = {}
    for r in pool.imap_unordered(_tensor, jobs, chunksize=1):
        res[r["i"]] = r
    return [res[j["i"]] for j in jobs]


def _sha(b: bytes) -> str:
    return hashlib.sha256(b).hexdigest()


def _chunk_table(manifest: bytes, names, lens, res, tiny_bytes) -> np.ndarray:
    """The publisher's chunk-digest table in manifest item order: big items
    chunked as they are, a group chunked over its packed staging."""
    items = O.ref_manifest_items(manifest)
    _ng, group_of, offset = O.assemble(lens)
    parts = []
    for is_group, index, length, _digest, _off in items:
        if not is_group:
            parts.append(res[int(index)]["chunks"])
            continue
        staging = np.zeros(int(length), np.uint8)
        for e in range(len(names)):
            if group_of[e] == int(index):
                b = tiny_bytes[e].view(np.uint8).reshape(-1)
                staging[int(offset[e]):int(offset[e]) + b.nbytes] = b
        parts.append(O.chunk_digests([staging], CHUNK))
    return np.concatenate(parts)


def publish_case(workload, pool, cast=False):
    """A single-shard replica of `workload` (seeds 42 + i), as bench.py
    publishes it: the reference manifest, the chunk table, per-tensor
    digests (and of the e4m3 cast)."""
    shapes = B.workload_shapes(workload)
    names = [n for n, _ in shapes]
    jobs = [{"i": i, "seed": 42 + i, "shape": s, "chunks": True, "cast": cast}
            for i, (_, s) in enumerate(shapes)]
    t0 = time.time()
    res = _run(jobs, pool)
    lens = [2 * _numel(s) for _, s in shapes]
    tiny = {i: r["bytes"] for i, r in enumerate(res) if "bytes" in r}
    man = O.ref_build_manifest_pre(names, lens, [r["digest"] for r in res], tiny)
    table = _chunk_table(man, names, lens, res, tiny)
    items = O.ref_manifest_items(man)
    out = {
        "workload": workload, "tensors": len(shapes), "bytes": int(sum(lens)),
        "manifest_sha256": _sha(man), "manifest_len": len(man),
        "items": int(items.shape[0]),
        "item_digests": ["%016X" % int(d) for d in items[:, 3]],
        "chunk_table_sha256": _sha(table.astype("<u8").tobytes()), "chunks": int(table.size),
        "tensor_digests": ["%016X" % r["digest"] for r in res],
    }
    if cast:
        out["cast_digests"] = ["%016X" % r["cast_digest"] for r in res]
    print(f"[golden] {workload}: {len(shapes)} tensors, {out['items']} items, "
          f"{out['chunks']} chunks, {time.time() - t0:.0f} s", flush=True)
    return out


def reshard_case(pool, fsdp=8, tp=2):
    """Config 3 as bench.py --reshard fsdp_tp2 builds it: full Qwen2.5-32B
    tensors (seeds 42 + i); trainer shard k holds row block k of every
    tensor (FSDP Shard(0)); reader shard s the TP-2 slice (tp_dim)."""
    shapes = B.workload_shapes("qwen25_32b")
    names = [n for n, _ in shapes]
    jobs = []
    for i, (n, s) in enumerate(shapes):
        sl = {f"f{k}": B.tp_slice(s, 2, 0, fsdp, k) for k in range(fsdp)}
        sl.update({f"r{k}": B.tp_slice(s, 2, B.tp_dim(n), tp, k) for k in range(tp)})
        jobs.append({"i": i, "seed": 42 + i, "shape": s, "slices": sl})
    t0 = time.time()
    res = _run(jobs, pool)
    trainer = []
    for k in range(fsdp):
        lens = []
        for n, s in shapes:
            g = B.tp_slice(s, 2, 0, fsdp, k)
            lens.append(g[3] * g[5])
        tiny = {i: r[f"f{k}_bytes"] for i, r in enumerate(res) if f"f{k}_bytes" in r}
        man = O.ref_build_manifest_pre(names, lens, [r[f"f{k}"] for r in res], tiny)
        trainer.append({"manifest_sha256": _sha(man), "manifest_len": len(man),
                        "items": int(O.ref_manifest_items(man).shape[0])})
    out = {"workload": "qwen25_32b", "fsdp": fsdp, "tp": tp, "tensors": len(shapes),
           "trainer_shards": trainer,
           "reader_slice_digests": [["%016X" % r[f"r{k}"] for r in res] for k in range(tp)]}
    print(f"[golden] qwen25_32b FSDP-{fsdp} -> TP-{tp}: {time.time() - t0:.0f} s", flush=True)
    return out


def main():
    assert O.ref_available(), "build oracle/_ref first (make -C oracle ref)"
    with Pool(min(8, os.cpu_count() or 1)) as pool:
        out = {
            "source": "tests/golden/make_scale_golden.py: reference digest64 / build_publish_payload "
                      "(oracle/_ref) over the bench's synthetic bytes; chunk partition, TP/FSDP "
                      "slices and the e4m3 cast restated by oracle/ros_oracle.c",
            "chunk_bytes": CHUNK,
            "config2_llama3_8b": publish_case("llama3_8b", pool),
            "config5_llama3_70b_tp8": publish_case("llama3_70b_tp8", pool, cast=True),
            "config3_qwen25_32b": reshard_case(pool),
        }
    with open(os.path.join(HERE, "scale.json"), "w") as f:
        json.dump(out, f, indent=1)
        f.write("\n")


if __name__ == "__main__":
    main()
