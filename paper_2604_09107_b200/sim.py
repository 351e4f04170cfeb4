"""Plan regression harness: the reference's SimNetwork
(transport_sim.cpp) moves modeled bytes with per-link delays; here a plan --
the registry's actual assignments -- is run through a fluid model of an
NVSwitch box whose constants are the B200 measurements in profiles/r1/, so
a planner change that would cost bandwidth shows up on a CPU.

Model (per GPU, one NVSwitch port):
  * a GPU that only sends or only receives moves `nvlink_one_way` bytes/s in
    that direction; a GPU doing both moves `nvlink_both_ways` each way
    (tools/nvlink_dir_probe.py: SM pulls 770-785 one way, ~672 both;
    tools/bidir_counters.sh: with both directions busy the receive lane
    carries 874-887 of 900 GB/s and the pull lands 679-691 of user data);
  * concurrent flows through one GPU port share it equally;
  * a reader chasing a source that is still filling cannot run ahead of it;
  * a GPU-local source is bound by HBM (read + write of every byte);
  * a host (retention offload) source by PCIe.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional


@dataclass
class LinkModel:
    nvlink_one_way: float = 785e9   # bytes/s, one direction busy (profiles/r1/nvlink_dir_v*.json)
    nvlink_both_ways: float = 672e9  # bytes/s per direction, both busy
    hbm: float = 6544e9             # bytes/s, measured copy (MEASURED_PEAKS.json)
    hbm_efficiency: float = 0.999   # fused copy+verify+watermarks vs a plain copy (bench N=1)
    pcie: float = 54.9e9            # bytes/s, pull from pinned host memory: copy-engine frames
                                    # verified in place (tools/offload_probe.py)


@dataclass
class Flow:
    reader: str
    source: str
    nbytes: int
    reader_gpu: int
    source_gpu: Optional[int]  # None: host memory (an offload)
    rate: float = 0.0
    seconds: float = 0.0
    upstream: list = field(default_factory=list)


def simulate(flows: list[Flow], model: LinkModel = LinkModel(), chasing: bool = True) -> list[Flow]:
    """Fill in each flow's steady rate and completion time."""
    sends, recvs = {}, {}
    for f in flows:
        if f.source_gpu is not None and f.source_gpu != f.reader_gpu:
            sends.setdefault(f.source_gpu, []).append(f)
            recvs.setdefault(f.reader_gpu, []).append(f)
    both = set(sends) & set(recvs)

    def port(g):
        return model.nvlink_both_ways if g in both else model.nvlink_one_way

    by_reader = {f.reader: f for f in flows}
    for f in flows:
        if f.source_gpu is None:
            cap = model.pcie
        elif f.source_gpu == f.reader_gpu:
            cap = model.hbm * model.hbm_efficiency / 2  # read + write in one HBM
        else:
            cap = min(port(f.source_gpu) / len(sends[f.source_gpu]),
                      port(f.reader_gpu) / len(recvs[f.reader_gpu]))
        f.rate = cap
    if chasing:  # a chaser runs no faster than what it chases
        changed = True
        while changed:
            changed = False
            for f in flows:
                up = by_reader.get(f.source)
                if up is not None and up.rate < f.rate:
                    f.rate = up.rate
                    changed = True
    for f in flows:
        f.seconds = f.nbytes / f.rate
        up = by_reader.get(f.source)
        if chasing and up is not None:
            f.seconds = max(f.seconds, up.nbytes / up.rate)
    return flows


def flows_from_plan(assigns, placement: dict, nbytes: dict, version: Optional[int] = None) -> list[Flow]:
    """Flows of a registry plan (ros.Cluster.assigns() / DistCluster.assigns()):
    `placement` maps a replica name to its GPU (None for a host offload),
    `nbytes` a reader to the bytes it lands."""
    out, seen = [], set()
    for a in assigns:
        if version is not None and a.version != version:
            continue
        if a.replica in seen:  # the latest assignment of a reader wins
            out = [f for f in out if f.reader != a.replica]
        seen.add(a.replica)
        out.append(Flow(a.replica, a.src, nbytes[a.replica], placement[a.replica],
                        placement.get(a.src)))
    return out


def per_receiver_gbs(flows: list[Flow]) -> dict:
    return {f.reader: f.nbytes / f.seconds / 1e9 for f in flows}
