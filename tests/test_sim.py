"""Plan regression harness: the registry's plans run
through the measured NVSwitch fluid model (paper_2604_09107_b200/sim.py) on
CPU.  The model is pinned to the B200 measurements in profiles/r1/ (each
case below cites the bench line it reproduces), then used to check the
planner: the 7-reader chain keeps every receiver at the two-direction port
rate, and a plan that fans every reader out of the trainer would not."""
import ctypes as C

import pytest

from paper_2604_09107_b200._lib import lib
from paper_2604_09107_b200.ros import Cluster
from paper_2604_09107_b200.sim import Flow, LinkModel, flows_from_plan, per_receiver_gbs, simulate
from tests.test_reshard import _open

LLAMA = 16_060_522_496
SHARD = 8_030_527_488


def _close(x, want, tol=0.06):
    return abs(x - want) <= tol * want


@pytest.mark.parametrize("case", [
    # (flows, measured per-receiver GB/s, source log)
    ([("r1", "t", LLAMA, 1, 0)], [785], "bench_c2_n2.log"),
    ([("r1", "t", LLAMA, 1, 0), ("r2", "r1", LLAMA, 2, 1), ("r3", "r2", LLAMA, 3, 2)],
     [678, 666, 653], "bench_c2_n4.log"),
    ([("a", "t", SHARD, 1, 0), ("b", "t", SHARD, 2, 0)], [394, 394], "bench_tp2_fanout_n3.log"),
    ([("r0", "t0", 17_640_734_720, 1, 0), ("r1", "t1", 17_640_734_720, 0, 1)], [673, 665],
     "bench_c5_ring_n2.log"),
])
def test_model_reproduces_measured_plans(case):
    spec, measured, log = case
    flows = simulate([Flow(r, s, n, rg, sg) for r, s, n, rg, sg in spec])
    got = [f.nbytes / f.seconds / 1e9 for f in flows]
    for g, m in zip(got, measured):
        assert _close(g, m), (log, got, measured)


def test_local_pull_is_hbm_bound():
    f = simulate([Flow("r", "t", LLAMA, 0, 0)])[0]
    # bench N=1: 4.92 ms kernel for the Llama-3-8B local pull (profiles/r1/final/bench_n1.log)
    assert _close(f.seconds * 1e3, 4.92, tol=0.05)


def test_offload_source_is_pcie_bound():
    f = simulate([Flow("r", "t+offload@1", LLAMA, 0, None)])[0]
    assert _close(f.nbytes / f.seconds / 1e9, 54.9, tol=0.02)  # tools/offload_probe.py, bench N=1 e2e


def _plan_of_simultaneous_readers(oracle, n_readers):
    from tests.test_retention import _manifest, _publish
    cl = Cluster()
    _open(cl, "trainer", 1, "")
    assert _publish(cl, "trainer", 1, _manifest(oracle, 1)) == 0
    readers = [f"rollout{i}" for i in range(1, n_readers + 1)]
    for r in readers:
        _open(cl, r, 1, "")
    for r in readers:
        assert lib.rs_server_replicate(cl.h, b"m", r.encode(), b"latest") == 0
    a = cl.assigns()
    cl.close()
    return readers, a


def test_planner_chain_keeps_every_receiver_at_port_rate(oracle):
    """The registry's plan for 7 simultaneous readers (the reference's
    chain) on 8 GPUs: every receiver lands at the two-direction port rate;
    the last one, which only receives, is capped by what it chases."""
    readers, assigns = _plan_of_simultaneous_readers(oracle, 7)
    placement = {"trainer": 0, **{r: i + 1 for i, r in enumerate(readers)}}
    flows = flows_from_plan(assigns, placement, {r: LLAMA for r in readers}, version=1)
    assert [(f.reader, f.source) for f in flows] == [
        (r, "trainer" if i == 0 else readers[i - 1]) for i, r in enumerate(readers)]
    rx = per_receiver_gbs(simulate(flows))
    m = LinkModel()
    assert all(_close(v, m.nvlink_both_ways / 1e9, tol=0.01) for v in rx.values()), rx


def test_fan_out_of_the_trainer_would_cost_bandwidth():
    """The counterfactual the planner avoids: seven readers all pulling the
    trainer share its port and land at a seventh of the rate."""
    flows = simulate([Flow(f"r{i}", "trainer", LLAMA, i, 0) for i in range(1, 8)])
    rx = per_receiver_gbs(flows)
    assert all(v < 120 for v in rx.values()), rx
