"""The drop-in boundary proven from the reference side.

integration/ref_scenarios.cpp compiles the reference-side adapters
(integration/refstore_b200/: level A B200Client over the C ABI, level B
B200Transport as the reference's DataTransport) against the UNMODIFIED
reference headers and links them with the reference library built from its
own sources (oracle/_ref) and libros_b200.so.  It then runs the reference's
client scenarios (tests/unit/test_client_core.cpp:163-202 and :346-377) on
the GPU and checks the reference's own counters; level C points the
reference's own data-plane dialer (StreamData) at the B200 process's TCP
server, which answers the reference wire (RSDP): items_verified == 3,
bytes_pulled exact, checksum_failures == 0 (2 + one report for the corrupt
source), bytes identical.

CPU: the binary builds (here, where /root/reference exists) and lists its
scenarios without a GPU.  GPU: every scenario passes."""
import os
import subprocess

import pytest

from tests.conftest import ROOT

BIN = os.path.join(ROOT, "integration", "_build", "ref_scenarios")
SCENARIOS = ["A replicate_pulls_bytes_that_verify", "B replicate_pulls_bytes_that_verify",
             "B corrupt_source_quiet_retry_report_repick", "A update_no_change_then_newer",
             "B update_no_change_then_newer", "B silent_source_reported_and_pull_moves",
             "B transport_equivalence_mem_vs_b200", "C rsdp_reference_reader_pulls_and_verifies",
             "A cross_link_update_fills_a_host_seed_then_consumes_it"]


def _binary():
    if os.path.isdir("/root/reference/proj/include"):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "ref"], check=True)
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "integration")], check=True)
    if not os.path.exists(BIN):
        pytest.skip("integration/_build/ref_scenarios not built (needs /root/reference headers)")
    return BIN


def test_reference_side_adapters_build_and_list():
    r = subprocess.run([_binary(), "--list"], capture_output=True, text=True, timeout=60)
    assert r.returncode == 0, r.stderr
    assert r.stdout.split("\n")[:len(SCENARIOS)] == SCENARIOS


@pytest.mark.gpu
def test_reference_scenarios_through_the_b200_path():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    r = subprocess.run([_binary()], capture_output=True, text=True, timeout=600)
    lines = [x for x in r.stdout.splitlines() if x.startswith(("PASS", "FAIL"))]
    assert r.returncode == 0, r.stdout + r.stderr
    assert [" ".join(x.split()[1:3]) for x in lines] == SCENARIOS
    kv = {" ".join(x.split()[1:3]): dict(f.split("=") for f in x.split()[3:]) for x in lines}
    for name in SCENARIOS[:2]:
        assert kv[name]["items_verified"] == "3"
        assert kv[name]["bytes_pulled"] == str((3 << 20) + 1000 + 2000 + 4096)
        assert kv[name]["checksum_failures"] == "0"
    assert int(kv[SCENARIOS[1]]["device_pulls"]) > 0
    assert int(kv[SCENARIOS[1]]["device_bytes"]) == 3 << 20  # the big item, moved by the kernel
    assert kv[SCENARIOS[2]]["checksum_failures"] == "2" and kv[SCENARIOS[2]]["failure_reports"] == "1"
    # the reference's StreamData over the B200 server's RSDP: 3 items verified
    assert kv[SCENARIOS[7]]["items_verified"] == "3"
    assert kv[SCENARIOS[7]]["bytes_pulled"] == str((3 << 20) + 1000 + 2000 + 4096)
    assert int(kv[SCENARIOS[5]]["failure_reports"]) >= 1
    assert int(kv[SCENARIOS[6]]["device_bytes"]) > 0
    # test_client_core.cpp:460-503 through B200Client: only the seed fill
    # crossed the link, the consumption was a local copy
    assert kv[SCENARIOS[8]] == {"bytes_pulled_cross_dc": "300000", "bytes_copied_local": "300000"}
