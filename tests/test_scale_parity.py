"""GPU: parity at BASELINE config scale, against the reference.

tests/golden/scale.json holds what the reference computes over the bench's
synthetic workloads (make_scale_golden.py: reference digest64 and
build_publish_payload over the bytes; chunk partition, TP/FSDP slices and the
e4m3 cast restated by the oracle).  Here the same workloads are generated on
the device (rs_synth_bf16, bit-exact with the oracle's generator), published
and pulled through the C ABI exactly as bench.py lays them out, and then:

* the publisher's manifest -- entry digests, packing, group digest, encoding
  -- is byte-identical to the reference's (sha256 of the bytes);
* the chunk-digest table equals the restatement's (sha256);
* every landed tensor's reference digest64 (computed on the device by K6,
  itself pinned to the reference's digest vectors) equals the reference's
  digest of the expected bytes: the tensor itself, its e4m3 cast, or its
  TP-2 slice.

Config 2: Llama-3-8B (16.06 GB), trainer -> reader on one GPU.
Config 5: the Llama-3-70B TP-8 shard (17.64 GB bf16) landed as e4m3.
Config 3: Qwen2.5-32B (65.5 GB) FSDP-8 trainer -> TP-2 reader, on one GPU.
"""
import hashlib
import json

import numpy as np
import pytest

from tests.conftest import golden

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def scale():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    with open(golden("scale.json")) as f:
        return json.load(f)


def _sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).astype("<u8").tobytes()).hexdigest()


def _hex(xs):
    return ["%016X" % x for x in xs]


def _pair(workload, reshard=False, cast=False, early=False):
    import bench as B
    from paper_2604_09107_b200.ros import Cluster
    dev = torch.device("cuda:0")
    shapes = B.workload_shapes(workload)
    tarena, tviews = B.alloc_replica(shapes, dev, seed_base=42)
    rarena, rviews = B.alloc_replica(shapes, dev, elem=1 if cast else 2)
    torch.cuda.synchronize()
    cl = Cluster()
    t = cl.open("m", "trainer", 8 if reshard else 1, early_publish=early)
    r = cl.open("m", "rollout1", 2 if reshard else 1)
    rslices = B.register_pair(t, r, shapes, tviews, rviews, dev, reshard, cast)
    return shapes, cl, t, r, tviews, rviews, rslices


def _free(*objs):
    torch.cuda.synchronize()
    for o in objs:
        if hasattr(o, "close"):
            o.close()
    torch.cuda.empty_cache()


@pytest.mark.parametrize("early", [False, True], ids=["reference_order", "early_publish"])
def test_config2_llama3_8b_matches_reference(scale, early):
    """early_publish: readers pull while the big-entry digests run; the
    manifest committed afterwards must still be the reference's bytes."""
    from paper_2604_09107_b200 import ros
    from paper_2604_09107_b200.ros import Status
    g = scale["config2_llama3_8b"]
    shapes, cl, t, r, tviews, rviews, _ = _pair("llama3_8b", early=early)
    try:
        assert sum(v.numel() for _, v in tviews) == g["bytes"] == 16_060_522_496
        assert t.publish(1).status == Status.ok
        if early:
            assert t.publish_pending
            res = r.replicate("latest")  # before the digests are in
            assert res.status == Status.ok, res
        man = t.manifest(0)
        assert len(man) == g["manifest_len"]
        assert hashlib.sha256(man).hexdigest() == g["manifest_sha256"]
        assert _sha(t.chunk_digests(0)) == g["chunk_table_sha256"]
        if not early:
            res = r.replicate("latest")
        assert res.status == Status.ok and res.version == 1, res
        assert r.manifest(0) == man
        table = r.chunk_digests(0)
        assert table.size == g["chunks"] and _sha(table) == g["chunk_table_sha256"]
        st = r.stats()
        assert st.items_verified == g["items"] == 227 and st.checksum_failures == 0
        got = ros.digest_spans([v.data_ptr() for _, v in rviews], [v.numel() for _, v in rviews])
        assert _hex(got) == g["tensor_digests"]
    finally:
        _free(cl)


def test_config5_llama3_70b_tp8_cast_matches_reference(scale):
    from paper_2604_09107_b200 import ros
    from paper_2604_09107_b200.ros import Status
    g = scale["config5_llama3_70b_tp8"]
    shapes, cl, t, r, tviews, rviews, _ = _pair("llama3_70b_tp8", cast=True)
    try:
        assert sum(v.numel() for _, v in tviews) == g["bytes"]
        assert t.publish(1).status == Status.ok
        assert hashlib.sha256(t.manifest(0)).hexdigest() == g["manifest_sha256"]
        res = r.replicate("latest")
        assert res.status == Status.ok, res
        # verified on the bf16 bytes the trainer published, landed as e4m3
        assert _sha(r.chunk_digests(0)) == g["chunk_table_sha256"]
        got = ros.digest_spans([w.data_ptr() for _, w in rviews], [w.numel() for _, w in rviews])
        assert _hex(got) == g["cast_digests"]
    finally:
        _free(cl)


def test_config3_qwen_fsdp8_to_tp2_matches_reference(scale):
    from paper_2604_09107_b200 import ros
    from paper_2604_09107_b200.ros import Status
    g = scale["config3_qwen25_32b"]
    shapes, cl, t, r, tviews, rviews, rslices = _pair("qwen25_32b", reshard=True)
    try:
        assert t.publish(1).status == Status.ok
        for k, want in enumerate(g["trainer_shards"]):
            assert hashlib.sha256(t.manifest(k)).hexdigest() == want["manifest_sha256"], k
        res = r.replicate("latest")
        assert res.status == Status.ok, res
        names = [n for n, _ in shapes]
        for s in range(2):
            bufs = [rslices[(s, n)][0] for n in names]
            got = ros.digest_spans([b.data_ptr() for b in bufs], [b.numel() for b in bufs])
            bad = [n for n, x, y in zip(names, _hex(got), g["reader_slice_digests"][s]) if x != y]
            assert not bad, (s, bad[:5])
    finally:
        _free(cl)
