"""GPU: the sm_100a kernels against the CPU oracle (bit-exact)."""
import json

import numpy as np
import pytest

from tests.conftest import golden

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")


def to_dev(arr: np.ndarray, dev, pad=0, offset=0):
    """Upload bytes at a chosen byte offset inside a fresh allocation."""
    raw = torch.zeros(arr.nbytes + offset + pad + 64, dtype=torch.uint8, device=dev)
    raw[offset:offset + arr.nbytes] = torch.from_numpy(arr.view(np.uint8).copy()).to(dev)
    return raw, raw.data_ptr() + offset


def test_synth_matches_oracle(dev, oracle):
    from paper_2604_09107_b200 import ros
    for seed, n, first in [(42, 1000, 0), (43, 4097, 0), (44, 77, 13), (45, 1 << 20, 5)]:
        t = torch.empty(n, dtype=torch.bfloat16, device=dev)
        ros.synth_bf16(t, seed, first)
        got = t.view(torch.int16).cpu().numpy().view(np.uint16)
        assert np.array_equal(got, oracle.synth_bf16(seed, n, first)), (seed, n, first)


def test_span_digests_match_reference_vectors(dev, oracle):
    from paper_2604_09107_b200 import ros
    g = json.load(open(golden("ref_digests.json")))["digests"]
    data = np.frombuffer(oracle.splitmix_bytes(99, 70000), np.uint8)
    for offset in (0, 1, 3, 8):
        raw, base = to_dev(data, dev, offset=offset)
        lens = [int(n) for n in g]
        got = ros.digest_spans([base] * len(lens), lens, 0)
        for n, d in zip(lens, got):
            assert d == int(g[str(n)], 16), (offset, n)


def test_span_digests_frozen_vectors(dev):
    from paper_2604_09107_b200 import ros
    v = json.load(open(golden("digest_vectors.json")))
    for s, want in v["strings"].items():
        arr = np.frombuffer(s.encode() or b"\0", np.uint8)
        raw, base = to_dev(arr, dev)
        assert ros.digest_spans([base], [len(s)], 0)[0] == int(want, 16)


def test_span_digests_large_and_many(dev, oracle):
    from paper_2604_09107_b200 import ros
    rng = np.random.default_rng(3)
    lens = [int(x) for x in rng.integers(1, 300000, 40)] + [64 << 20]
    bufs = [torch.randint(0, 256, (n,), dtype=torch.uint8, device=dev) for n in lens]
    got = ros.digest_spans([b.data_ptr() for b in bufs], lens, 0)
    for b, d in zip(bufs, got):
        assert d == oracle.xxh64(b.cpu().numpy())


@pytest.mark.parametrize("chunk", [256, 4096, 4112, 65536])
def test_pull_spans_copy_and_chunk_digests(dev, oracle, chunk):
    from paper_2604_09107_b200 import ros
    rng = np.random.default_rng(chunk)
    lens = [1, 15, 16, 17, 31, 32, 33, 255, 256, 257, 4095, 4096, 4097, 100003, 3 << 20, 777]
    srcs = [torch.randint(0, 256, (n,), dtype=torch.uint8, device=dev) for n in lens]
    # destinations at assorted alignments
    dst_raw = [torch.zeros(n + 32, dtype=torch.uint8, device=dev) for n in lens]
    offs = [int(x) for x in rng.integers(0, 17, len(lens))]
    dsts = [d.data_ptr() + o for d, o in zip(dst_raw, offs)]
    want = oracle.chunk_digests([s.cpu().numpy() for s in srcs], chunk)
    out = torch.zeros(len(want), dtype=torch.int64, device=dev)
    code, ms = ros.pull_spans([s.data_ptr() for s in srcs], dsts, lens, chunk, None, out, 0)
    torch.cuda.synchronize()
    assert code == 0
    assert np.array_equal(out.cpu().numpy().view(np.uint64), want)
    for s, d, o, n in zip(srcs, dst_raw, offs, lens):
        assert torch.equal(d[o:o + n], s)
        assert int(d[:o].abs().sum()) == 0 and int(d[o + n:].abs().sum()) == 0  # no overrun
    # verification against the correct table passes; a corrupted one fails
    expect = torch.from_numpy(want.view(np.int64).copy()).to(dev)
    code, _ = ros.pull_spans([s.data_ptr() for s in srcs], dsts, lens, chunk, expect, None, 0)
    assert code == 0
    expect[len(want) // 2] ^= 1
    code, _ = ros.pull_spans([s.data_ptr() for s in srcs], dsts, lens, chunk, expect, None, 0)
    assert code == 1  # kPullChecksum after the quiet retry


def test_pull_spans_misaligned_sources(dev, oracle):
    from paper_2604_09107_b200 import ros
    data = np.frombuffer(oracle.splitmix_bytes(5, 50000), np.uint8)
    for off in (1, 2, 4, 8, 12):
        raw, base = to_dev(data, dev, offset=off)
        dst = torch.zeros(data.nbytes, dtype=torch.uint8, device=dev)
        want = oracle.chunk_digests([data], 4096)
        out = torch.zeros(len(want), dtype=torch.int64, device=dev)
        code, _ = ros.pull_spans([base], [dst.data_ptr()], [data.nbytes], 4096, None, out, 0)
        assert code == 0
        assert np.array_equal(dst.cpu().numpy(), data)
        assert np.array_equal(out.cpu().numpy().view(np.uint64), want)


def test_pull_spans_empty(dev):
    from paper_2604_09107_b200 import ros
    code, _ = ros.pull_spans([], [], [], 4096, None, None, 0)
    assert code == 0


def test_e4m3_all_bf16_patterns(dev, oracle):
    from paper_2604_09107_b200 import ros
    pat = np.arange(65536, dtype=np.uint32).astype(np.uint16)
    src = torch.from_numpy(pat.view(np.int16).copy()).to(dev)
    dst = torch.zeros(65536, dtype=torch.uint8, device=dev)
    ros.bf16_to_e4m3(src, dst)
    got = dst.cpu().numpy()
    want = oracle.bf16_to_e4m3(pat)
    # bit-exact on every pattern, NaNs included (both give 0x7F)
    assert np.array_equal(got, want)


def test_ldg_kernel_variant_still_bit_exact(dev):
    """The LDGSTS (non-TMA) pull kernel, selected with RSB_PULL_KERNEL=ldg,
    passes the same copy/digest parity tests."""
    import os
    import subprocess
    import sys
    from tests.conftest import ROOT
    env = dict(os.environ, RSB_PULL_KERNEL="ldg")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-m", "gpu", "-x",
                        "tests/test_gpu_kernels.py", "-k", "pull_spans"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
