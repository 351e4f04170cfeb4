"""Pull schedule order (pullplan.cpp schedule_order), host logic on CPU.

The order lists the batches some segment touches; with sources behind more
than one link (ItemDesc.pad = link class) it interleaves the classes in
proportion to their batch counts, each class front to back.  An empty
result means "every batch, in batch order"."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_2604_09107_b200", "csrc")


@pytest.fixture(scope="module")
def run(tmp_path_factory):
    gxx = shutil.which("g++")
    if gxx is None:
        pytest.skip("g++ not found")
    inc = "/usr/local/cuda/include"
    exe = str(tmp_path_factory.mktemp("so") / "schedule_order")
    cmd = [gxx, "-std=c++17", "-O1", "-I", CSRC, "-I", inc,
           os.path.join(ROOT, "tests", "cpp", "schedule_order_main.cpp"),
           os.path.join(CSRC, "pullplan.cpp"), "-o", exe,
           "-L/usr/local/cuda/lib64", "-lcudart_static", "-lpthread", "-ldl", "-lrt"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        pytest.fail(r.stderr[-2000:])

    def go(cases, env=None):
        txt = ""
        for nb, segs in cases:
            txt += f"{nb} {len(segs)}\n" + "".join(f"{c0} {cl} {ln} {cls}\n" for c0, cl, ln, cls in segs)
        out = subprocess.run([exe], input=txt, capture_output=True, text=True,
                             env={**os.environ, **(env or {})}, check=True).stdout.split("\n")
        return [[int(x) for x in line.split()[1:]] for line in out if line]
    return go


def test_one_link_every_batch_is_batch_order(run):
    # two items of 64 and 40 chunks (batch-aligned), both local
    assert run([(4, [(0, 4096, 64 * 4096, 0), (64, 4096, 40 * 4096, 0)])]) == [[]]


def test_untouched_batches_are_left_out(run):
    # a hash pass over items at batches 1 and 5..6 of an 8-batch payload
    (order,) = run([(8, [(32, 4096, 32 * 4096, 0), (160, 2560, 40 * 2560, 0)])])
    assert order == [1, 5, 6]


def test_two_links_interleave_in_proportion(run):
    # 12 local batches then 4 batches from a peer (class 2 + device 1 = 3)
    (order,) = run([(16, [(0, 4096, 12 * 32 * 4096, 0), (12 * 32, 4096, 4 * 32 * 4096, 3)])])
    assert sorted(order) == list(range(16))
    local = [b for b in order if b < 12]
    peer = [b for b in order if b >= 12]
    assert local == sorted(local) and peer == sorted(peer)  # each class front to back
    # at every prefix the classes have advanced by the same fraction (+- one batch)
    for k in range(1, 17):
        pre = order[:k]
        f_local = sum(b < 12 for b in pre) / 12
        f_peer = sum(b >= 12 for b in pre) / 4
        assert abs(f_local - f_peer) <= 1 / 4 + 1e-9, (k, pre)
    assert order[:4] == [0, 1, 12, 2]  # keys (r + 1/2) / n: ties go to the lower batch


def test_interleave_can_be_turned_off(run):
    segs = [(0, 4096, 12 * 32 * 4096, 0), (12 * 32, 4096, 4 * 32 * 4096, 3)]
    assert run([(16, segs)], env={"RSB_BATCH_ORDER": "0"}) == [[]]
