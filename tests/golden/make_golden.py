"""Generates tests/golden/*.json from the REFERENCE implementation.

Run here (needs /root/reference built into oracle/_ref by ``make -C oracle``):

    python tests/golden/make_golden.py

Every value below comes from the unmodified reference refstore library
(oracle/_ref/librefstore_ref.so) -- its digest64, assemble_manifest/
pack_group/encode and its ServerCore planner driven through ClientCore +
MemNetwork + SimExecutor exactly like the reference's ClusterFix
(tests/unit/test_client_core.cpp:23-117).  The frozen XXH64 vectors are the
reference's own (tests/unit/test_digest.cpp:42-69).  The committed fixtures
let the GPU box (where /root/reference does not exist) check parity.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402

from tests.golden.models import llama3_8b, tiny_set  # noqa: E402


def frozen_digest_vectors() -> dict:
    # test_digest.cpp:42-45, 54-59, 68-69 (values copied verbatim)
    return {
        "source": "/root/reference/proj/tests/unit/test_digest.cpp:42-69",
        "strings": {"": "EF46DB3751D8E999", "a": "D24EC4F1A98C6E5B", "abc": "44BC2CF5AD770999",
                    "Hello, world!": "F58336A78B6F9476"},
        "pattern": {"3": "C2D5FE9E5E827296", "4": "6F20103DC53D2B38", "7": "DBCF5F2C174ED056",
                    "8": "FFB16F759C44D7C3", "15": "C959035ACD9D294B", "16": "6AAEBC48FDDBE290",
                    "31": "C55294C726A80342", "32": "0FACD3340FF96628", "33": "851A6EA9CBE767AB",
                    "63": "AD40449420FCEAC3", "64": "342FC0C8324C6C58"},
        "splitmix": [{"seed": 1, "n": 1024, "digest": "2CED67D3BBC7413B"},
                     {"seed": 7, "n": 1 << 20, "digest": "2C74017032DC0470"}],
    }


def ref_digests_extra() -> dict:
    """Reference digest64 over lengths 0..300 of splitmix bytes + odd sizes."""
    out = {}
    data = O.splitmix_bytes(99, 70000)
    for n in list(range(0, 301)) + [1023, 1024, 1025, 4095, 4096, 4097, 65535, 65536, 69999]:
        out[str(n)] = "%016X" % O.ref_digest64(data[:n])
    return {"source": "oracle/_ref digest64 over splitmix_bytes(99, n)", "digests": out}


def manifests() -> dict:
    cases = {}
    # test_manifest.cpp:32-79 packing oracle (threshold 100, target 250)
    names = ["e0", "e1", "e2", "e3", "e4", "e5"]
    lens = [50, 200, 60, 70, 80, 30]
    dig = [1, 2, 3, 4, 5, 6]
    cases["packing_oracle"] = {"names": names, "lens": lens, "digests": dig, "tiny": 100,
                               "target": 250, "seal": False,
                               "encoded": O.ref_assemble_manifest(names, lens, dig, 100, 250).hex(),
                               "items": O.ref_manifest_items(
                                   O.ref_assemble_manifest(names, lens, dig, 100, 250)).tolist()}
    # threshold edge (test_manifest.cpp:81-91)
    cases["threshold_edge"] = {"names": ["a", "b"], "lens": [100, 99], "digests": [1, 2], "tiny": 100,
                               "target": 250, "seal": False,
                               "encoded": O.ref_assemble_manifest(["a", "b"], [100, 99], [1, 2], 100,
                                                                  250).hex()}
    # 1000 x 1 MB default limits (test_manifest.cpp:93-105)
    nm = [f"t{i}" for i in range(1000)]
    enc = O.ref_assemble_manifest(nm, [1_000_000] * 1000, [0] * 1000)
    cases["thousand_1mb"] = {"names": nm, "lens": [1_000_000] * 1000, "digests": [0] * 1000,
                             "tiny": 2 << 20, "target": 64 << 20, "seal": False,
                             "sha256": hashlib.sha256(enc).hexdigest(), "n_bytes": len(enc),
                             "n_items": int(O.ref_manifest_items(enc).shape[0])}
    # Llama-3-8B inventory with modeled (version-1) digests, sealed groups.
    names, lens = llama3_8b()
    dig = [O.ref().ref_modeled_entry_digest(n.encode(), 1, l) for n, l in zip(names, lens)]
    enc = O.ref_assemble_manifest(names, lens, dig, seal=True)
    cases["llama3_8b_modeled"] = {"names": names, "lens": lens, "digests": dig,
                                  "tiny": 2 << 20, "target": 64 << 20, "seal": True,
                                  "sha256": hashlib.sha256(enc).hexdigest(), "n_bytes": len(enc),
                                  "n_items": int(O.ref_manifest_items(enc).shape[0])}
    # Real bytes: build_publish_payload over pattern-filled tensors.
    names, arrays = tiny_set()
    enc = O.ref_build_manifest(names, arrays)
    cases["tiny_set_real"] = {"names": names, "lens": [a.nbytes for a in arrays],
                              "encoded": enc.hex(), "items": O.ref_manifest_items(enc).tolist()}
    enc = O.ref_build_manifest(names, arrays, 100 << 10, 1 << 20)
    cases["tiny_set_real_small_limits"] = {"names": names, "lens": [a.nbytes for a in arrays],
                                           "tiny": 100 << 10, "target": 1 << 20,
                                           "encoded": enc.hex(),
                                           "items": O.ref_manifest_items(enc).tolist()}
    return cases


def plan(scenario: str) -> dict:
    """Runs a planner scenario on the reference (modeled payloads)."""
    c = O.RefCluster(threaded=False, server_pipeline=scenario != "pipeline_off")
    names, lens = tiny_set_sizes = (["w0", "w1", "w2"], [4 << 20, 1 << 20, 3000])
    reps = []
    if scenario in ("chain7", "pipeline_off"):
        reps = ["trainer"] + [f"rollout{i}" for i in range(1, 8)]
    elif scenario == "spread":
        reps = ["src1", "src2", "src3"] + [f"r{i}" for i in range(1, 7)]
    elif scenario == "parked":
        reps = ["dst1", "dst2", "src"]
    for r in reps:
        c.add(r, 1)
        for n, l in zip(names, lens):
            c.register_modeled(r, 0, n, l)
    events = []
    if scenario in ("chain7", "pipeline_off"):
        events.append(("publish", "trainer", 1, c.publish("trainer", 1)[0]))
        st, vs, _, _ = c.pull_many([f"rollout{i}" for i in range(1, 8)])
        events.append(("replicate_many", [f"rollout{i}" for i in range(1, 8)], st))
    elif scenario == "spread":
        events.append(("publish", "src1", 1, c.publish("src1", 1)[0]))
        st, _, _, _ = c.pull_many(["src2"])
        events.append(("replicate_many", ["src2"], st))
        st, _, _, _ = c.pull_many(["src3"])
        events.append(("replicate_many", ["src3"], st))
        st, _, _, _ = c.pull_many([f"r{i}" for i in range(1, 7)])
        events.append(("replicate_many", [f"r{i}" for i in range(1, 7)], st))
    elif scenario == "parked":
        # test_server_core.cpp:317-340: both readers park before any version
        # exists; src then publishes and they wake oldest-first.
        st = _pull_with_publish(c, ["dst1", "dst2"], "src")
        events.append(("parked_then_publish", ["dst1", "dst2"], st))
    c.settle()
    assigns = [a.__dict__ for a in c.assigns()]
    views = {r: c.view(r) for r in reps}
    c.close()
    return {"scenario": scenario, "replicas": reps, "tensors": list(zip(names, lens)),
            "events": events, "assigns": assigns, "views": views}


def _pull_with_publish(c, readers, src):
    """Issue replicate on readers (they park), then publish on src, then run."""
    import ctypes as C
    lib = c.lib
    n = len(readers)
    arr = (C.c_char_p * n)(*[r.encode() for r in readers])
    st = np.zeros(n, np.int32)
    lib.ref_cluster_publish_during.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_char_p,
                                               C.c_uint64, C.c_void_p]
    rc = lib.ref_cluster_publish_during(c.h, n, C.cast(arr, C.c_void_p), src.encode(), 1,
                                        st.ctypes.data)
    assert rc == 0
    return [int(x) for x in st]


def chunk_digests() -> dict:
    """Chunk digests over synthetic bf16 tensors: the reference digest64 applied
    to our chunk partition (chunk j of item i = bytes [j*C, min((j+1)*C, len)))."""
    out = {}
    for seed, n_elems, chunk in [(42, 1000, 256), (43, 4096, 4096), (44, 100003, 4096),
                                 (45, 5, 4096), (46, 65536, 65536)]:
        arr = O.synth_bf16(seed, n_elems).view(np.uint8)
        digs = []
        for off in range(0, arr.nbytes, chunk):
            digs.append("%016X" % O.ref_digest64(arr[off:off + chunk]))
        out[f"{seed}:{n_elems}:{chunk}"] = {"item_digest": "%016X" % O.ref_digest64(arr),
                                           "chunks": digs,
                                           "head_u16": [int(x) for x in O.synth_bf16(seed, 8)]}
    return {"source": "oracle/_ref digest64 over ro_synth_bf16 bytes", "cases": out}


def main():
    if not O.ref_available():
        raise SystemExit("build oracle/_ref first: make -C oracle")
    files = {
        "digest_vectors.json": frozen_digest_vectors(),
        "ref_digests.json": ref_digests_extra(),
        "manifests.json": manifests(),
        "plans.json": {s: plan(s) for s in ("chain7", "pipeline_off", "spread", "parked")},
        "chunk_digests.json": chunk_digests(),
    }
    for name, data in files.items():
        with open(os.path.join(HERE, name), "w") as f:
            json.dump(data, f, indent=1, sort_keys=True)
        print("wrote", name)


if __name__ == "__main__":
    main()
