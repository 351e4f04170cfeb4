"""GPU, one device: the kernel shape every chain hop runs, on the driver's
1-GPU box.

A plain peer pull (a chain hop over NVLink: identity segments, no cast) is
launched as V16 -- the V13 pipeline shape releasing every verified batch at
once -- and reads its source through per-lane bulk-copy slots instead of
tensor-map boxes (pull_tma.cu launch_pull_tma, pullplan.cpp peer segments).
On one GPU every source is local, so the library would pick V13 with boxes.
These runs force the hop's shape (RSB_TMA_VARIANT=16, RSB_NO_MAPS=1) and
repeat the copy/verify parity tests, the client scenarios and the chase
tests with it: the bytes, digests and outcomes must not change."""
import os
import subprocess
import sys

import pytest

from tests.conftest import ROOT

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("target", [
    ["tests/test_gpu_kernels.py", "-k", "pull_spans"],
    ["tests/test_gpu_chase.py"],
    ["tests/test_gpu_client.py"],
])
def test_chain_hop_shape_is_bit_exact(target):
    env = dict(os.environ, RSB_TMA_VARIANT="16", RSB_NO_MAPS="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-m", "gpu", "-x", *target],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert " passed" in r.stdout and " skipped" not in r.stdout, r.stdout[-2000:]
