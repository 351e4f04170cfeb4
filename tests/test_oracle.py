"""CPU: pin the oracle (our C restatement) to the reference's golden vectors
and to the reference library itself."""
import json

import numpy as np
import pytest

from tests.conftest import golden
from tests.golden.models import llama3_8b, tiny_set


def load(name):
    with open(golden(name)) as f:
        return json.load(f)


def test_frozen_xxh64_vectors(oracle):
    g = load("digest_vectors.json")  # test_digest.cpp:42-69
    for s, want in g["strings"].items():
        assert oracle.xxh64(s.encode()) == int(want, 16), s
    for n, want in g["pattern"].items():
        assert oracle.xxh64(oracle.pattern_bytes(int(n))) == int(want, 16), n
    for case in g["splitmix"]:
        assert oracle.xxh64(oracle.splitmix_bytes(case["seed"], case["n"])) == int(case["digest"], 16)


def test_xxh64_matches_reference_fixture(oracle):
    g = load("ref_digests.json")
    data = oracle.splitmix_bytes(99, 70000)
    for n, want in g["digests"].items():
        assert oracle.xxh64(data[:int(n)]) == int(want, 16), n


def test_xxh64_matches_reference_library_random(ref):
    rng = np.random.default_rng(7)
    for n in list(rng.integers(0, 5000, 50)) + [0, 31, 32, 33, 1 << 16]:
        b = rng.integers(0, 256, int(n), dtype=np.uint8)
        assert ref.xxh64(b) == ref.ref_digest64(b)


def test_packing_oracle(oracle):
    # test_manifest.cpp:32-79
    ng, g, off = oracle.assemble([50, 200, 60, 70, 80, 30], 100, 250)
    assert ng == 2
    assert list(g) == [0, -1, 0, 0, 1, 1]
    assert list(off) == [0, 0, 50, 110, 0, 80]
    # threshold edge (test_manifest.cpp:81-91)
    ng, g, _ = oracle.assemble([100, 99], 100, 250)
    assert ng == 1 and list(g) == [-1, 0]
    # 1000 x 1 MB -> 15 groups of 67/62 (test_manifest.cpp:93-105)
    ng, g, _ = oracle.assemble([1_000_000] * 1000)
    assert ng == 15
    counts = np.bincount(g[g >= 0])
    assert list(counts[:14]) == [67] * 14 and counts[14] == 62


def test_manifest_encode_matches_reference_fixtures(oracle):
    m = load("manifests.json")
    for key in ("packing_oracle", "threshold_edge"):
        c = m[key]
        ng, g, off = oracle.assemble(c["lens"], c["tiny"], c["target"])
        enc = oracle.manifest_encode(c["names"], c["lens"], c["digests"], g, off, ng, [0] * ng)
        assert enc.hex() == c["encoded"], key


def test_publish_manifest_real_bytes(oracle):
    m = load("manifests.json")
    names, arrays = tiny_set()
    assert oracle.publish_manifest(names, arrays).hex() == m["tiny_set_real"]["encoded"]
    c = m["tiny_set_real_small_limits"]
    assert oracle.publish_manifest(names, arrays, c["tiny"], c["target"]).hex() == c["encoded"]


def test_llama3_8b_inventory(oracle):
    names, lens = llama3_8b()
    assert len(names) == 291 and sum(lens) == 16_060_522_496
    ng, g, _ = oracle.assemble(lens)
    assert ng == 1 and int((g == 0).sum()) == 65
    items = 291 - 65 + 1
    assert items == 227
    assert load("manifests.json")["llama3_8b_modeled"]["n_items"] == 227


def test_chunk_digests_and_synth(oracle):
    g = load("chunk_digests.json")["cases"]
    for key, case in g.items():
        seed, n, chunk = map(int, key.split(":"))
        arr = oracle.synth_bf16(seed, n)
        assert [int(x) for x in arr[:8]] == case["head_u16"][:min(n, 8)]
        assert oracle.xxh64(arr) == int(case["item_digest"], 16)
        got = oracle.chunk_digests([arr], chunk)
        assert ["%016X" % int(x) for x in got] == case["chunks"]


def test_synth_values_are_bf16_in_range(oracle):
    v = oracle.synth_bf16(42, 1 << 16)
    f = (v.astype(np.uint32) << 16).view(np.float32)
    # f32 in [-1, 1); RNE to bf16 can round the top end up to exactly 1.0
    assert np.all(np.isfinite(f)) and f.min() >= -1.0 and f.max() <= 1.0
    assert abs(float(f.mean())) < 0.02


@pytest.mark.parametrize("x,want", [
    (0.0, 0x00), (-0.0, 0x80), (1.0, 0x38), (-1.0, 0xB8), (448.0, 0x7E), (500.0, 0x7E),
    (1e30, 0x7E), (-1e30, 0xFE), (2.0 ** -9, 0x01), (2.0 ** -10, 0x00), (1.5 * 2 ** -10, 0x01),
    (0.015625, 0x08), (1.0625, 0x38), (1.1875, 0x3A), (float("inf"), 0x7E),
])
def test_e4m3_cast_definition(oracle, x, want):
    bf = (np.array([x], np.float32).view(np.uint32) >> 16).astype(np.uint16)
    assert int(oracle.bf16_to_e4m3(bf)[0]) == want


def test_e4m3_nan(oracle):
    assert int(oracle.bf16_to_e4m3(np.array([0x7FC0], np.uint16))[0]) == 0x7F


def test_scale_fixture_is_pinned_to_the_port(oracle):
    """tests/golden/scale.json (reference digests at BASELINE scale) agrees
    with the oracle's generator + XXH64 on the tensors small enough to redo
    here: the norms of Llama-3-8B and of the Llama-3-70B TP-8 shard (bytes
    and e4m3 cast)."""
    import json
    from tests.conftest import golden
    import bench as B
    g = json.load(open(golden("scale.json")))
    c2 = g["config2_llama3_8b"]
    assert c2["tensors"] == 291 and c2["items"] == 227 and c2["bytes"] == 16_060_522_496
    assert len(c2["item_digests"]) == 227 and c2["chunks"] == 3_921_026
    for key, cast in (("config2_llama3_8b", False), ("config5_llama3_70b_tp8", True)):
        shapes = B.workload_shapes(g[key]["workload"])
        for i, (n, s) in enumerate(shapes):
            if "norm" not in n or i % 7:
                continue
            a = oracle.synth_bf16(42 + i, s[0])
            assert "%016X" % oracle.xxh64(a) == g[key]["tensor_digests"][i], n
            if cast:
                assert "%016X" % oracle.xxh64(oracle.bf16_to_e4m3(a)) == g[key]["cast_digests"][i], n
    c3 = g["config3_qwen25_32b"]
    assert len(c3["trainer_shards"]) == 8 and len(c3["reader_slice_digests"]) == 2
