"""Benchmark of the B200 ROS read path (BASELINE.json metric: per-receiver pull
GB/s; weight-update latency).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload llama3_8b|config1] [--no-verify]

Workload (config.workload): BASELINE configs[1], Llama-3-8B bf16 weights
(291 tensors, 16,060,522,496 B, synthetic values of SURVEY.md §8d) published
by a trainer replica.  N=1: trainer and one reader on cuda:0, the pull runs
HBM->HBM on one GPU (bound: HBM).  N>1 (torchrun, one rank per GPU): rank 0
is the trainer, ranks 1..N-1 are readers planned by the registry (a chain,
like the reference planner); every reader pulls over NVLink (bound: ingress).

A step = one full weight update: every reader drops its copy
(unpublish + invalidate) and replicates "latest" through the C ABI --
registry plan, bind, the fused pull+verify kernel, group unpack, complete.
`value` = bytes landed by all readers / device time of the timed steps
(max over ranks).  `e2e` = the same metric over host wall-clock of the
rs_replicate calls (descriptor H2D + status D2H inside).  Inputs (16 GB per
replica) are far larger than the 126 MB L2, so no flush is needed.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "per-receiver pull GB/s"
UNIT = "GB/s"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ----------------------------------------------------------------- clocks
class ClockSampler:
    """SM clocks + throttle reasons sampled DURING the timed region through
    NVML (a poll every ~2 ms, so even a 30 ms region gets samples)."""
    REASONS = {  # nvmlClocksEventReason* bits
        "sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20,
        "hw_thermal_slowdown": 0x40,
    }

    def __init__(self, index: int):
        self.index = index
        self.samples: list[tuple[float, int]] = []
        self.smax = None
        self.err = None
        self._stop = threading.Event()
        self.t = None

    def start(self):
        try:
            import pynvml as N
            N.nvmlInit()
            self.N = N
            self.h = N.nvmlDeviceGetHandleByIndex(self.index)
            self.smax = float(N.nvmlDeviceGetMaxClockInfo(self.h, N.NVML_CLOCK_SM))
        except Exception as e:  # noqa: BLE001 - report, do not fail the bench
            self.err = f"nvml unavailable: {e}"
            return
        self.t = threading.Thread(target=self._run, daemon=True)
        self.t.start()

    def _run(self):
        N = self.N
        while not self._stop.is_set():
            try:
                sm = float(N.nvmlDeviceGetClockInfo(self.h, N.NVML_CLOCK_SM))
                rs = int(N.nvmlDeviceGetCurrentClocksEventReasons(self.h))
                self.samples.append((sm, rs))
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.002)

    def stop(self) -> dict:
        if self.t is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [self.err or "no sampler"]}
        self._stop.set()
        self.t.join(timeout=2)
        reasons = sorted({n for _, r in self.samples for n, b in self.REASONS.items() if r & b})
        sm = [x for x, _ in self.samples]
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": self.smax,
                "reasons": reasons, "samples": len(sm), "source": "nvml"}


class NvlinkCounters:
    """NVLink bytes this GPU sent / received, from NVML's per-link counters
    (NVML_FI_DEV_NVLINK_COUNT_XMIT_BYTES / _RCV_BYTES summed over the links;
    the aggregate THROUGHPUT_RAW_TX/RX fields in KiB as a fallback).  Raw
    link bytes: user data plus protocol, both directions of the port."""

    def __init__(self, index: int):
        self.err = None
        try:
            import pynvml as N
            N.nvmlInit()
            self.N = N
            self.h = N.nvmlDeviceGetHandleByIndex(index)
            self.links = [l for l in range(18) if self._up(l)]
        except Exception as e:  # noqa: BLE001 - report, do not fail the bench
            self.err = f"nvml unavailable: {e}"

    def _up(self, link):
        try:
            return self.N.nvmlDeviceGetNvLinkState(self.h, link) == self.N.NVML_FEATURE_ENABLED
        except Exception:  # noqa: BLE001
            return False

    def _fields(self, reqs):
        vals = self.N.nvmlDeviceGetFieldValues(self.h, reqs)
        out = []
        for v in vals:
            if v.nvmlReturn != 0:
                return None
            out.append(int(v.value.ullVal))
        return out

    def read(self):
        """(tx_bytes, rx_bytes, source) or None."""
        if self.err:
            return None
        N = self.N
        try:
            per = self._fields([(N.NVML_FI_DEV_NVLINK_COUNT_XMIT_BYTES, l) for l in self.links] +
                               [(N.NVML_FI_DEV_NVLINK_COUNT_RCV_BYTES, l) for l in self.links])
            if per is not None and self.links:
                k = len(self.links)
                return sum(per[:k]), sum(per[k:]), "nvml per-link XMIT/RCV bytes"
        except Exception:  # noqa: BLE001
            pass
        try:
            agg = self._fields([(N.NVML_FI_DEV_NVLINK_THROUGHPUT_RAW_TX, 0xFFFFFFFF),
                                (N.NVML_FI_DEV_NVLINK_THROUGHPUT_RAW_RX, 0xFFFFFFFF)])
            if agg is not None:
                return agg[0] * 1024, agg[1] * 1024, "nvml THROUGHPUT_RAW (KiB)"
        except Exception as e:  # noqa: BLE001
            self.err = str(e)
        return None


# NVLink 5 user-data bounds for SM-driven pulls, from the ncu nvlrx/nvltx
# counters of the pull kernel (profiles/r1/ncu_nvlink_counters.json): read
# responses add 12.5% protocol bytes on the wire, read requests 18.75% of the
# pulled bytes in the opposite direction.  One direction busy: 900/1.125;
# both directions busy (a chain's middle GPUs): 900/(1.125+0.1875).
NVL_RESP, NVL_REQ = 0.125, 0.1875
NVL_ONE_WAY = 900.0 / (1 + NVL_RESP)
NVL_BOTH_WAYS = 900.0 / (1 + NVL_RESP + NVL_REQ)


def measured_peaks() -> dict:
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return {"hbm_gbs": d.get("hbm_gbs", 6650.0), "src": "measured"}
    return {"hbm_gbs": 6650.0, "src": "fallback"}


def ncu_traffic(kind: str, user_bytes: int = 0, workload: str = None):
    """Per-launch bytes of the pull kernel from the committed ncu captures:
    DRAM bytes for a local pull ("local", "cast"); for a peer pull ("nvlink")
    the bytes the reader's NVLink port receives (user data + read-response
    protocol), scaled from the captured ratio to `user_bytes`."""
    p = os.path.join(ROOT, "profiles", "ncu_pull_summary.json")
    if not os.path.exists(p):
        return None
    try:
        with open(p) as f:
            d = json.load(f)
        if kind == "nvlink":
            r = d.get("nvlink", {}).get("link_rx_bytes_per_user_byte")
            return round(r * user_bytes) if r and user_bytes else None
        e = d.get(kind, {})
        if workload is not None and e.get("workload") not in (None, workload):
            return None  # captured on another workload
        return e.get("dram_bytes_per_launch")
    except (OSError, ValueError):
        return None


# --------------------------------------------------------------- workload
def workload_shapes(name: str):
    from tests.golden.models import config1, llama3_8b_shapes, llama3_70b_shapes
    if name == "llama3_8b":
        return llama3_8b_shapes()
    if name == "config1":
        return config1()
    if name == "big16":  # diagnostic: 16 x 512 MiB (the nvlink_dir_probe span set)
        return [(f"w{i}", (16384, 16384)) for i in range(16)]
    if name == "qwen25_32b":
        from tests.golden.models import qwen25_32b_shapes
        return qwen25_32b_shapes()
    if name == "llama3_70b_tp8":
        # config 5: one TP-8 shard (rank 0) of Llama-3-70B, each tensor's
        # slice contiguous as its trainer rank holds it
        out = []
        for n, shape in llama3_70b_shapes():
            d = tp_dim(n)
            if d is None:
                out.append((n, shape))
            elif d == 0:
                out.append((n, (shape[0] // 8,) + tuple(shape[1:])))
            else:
                out.append((n, (shape[0], shape[1] // 8)))
        return out
    raise SystemExit(f"unknown workload {name}")


def alloc_replica(shapes, dev, seed_base=None, elem=2):
    """One contiguous arena per replica, tensors as views (IPC-exportable);
    elem=1: an e4m3 landing arena (half the bytes, same layout)."""
    import torch

    from paper_2604_09107_b200 import ros
    sizes = [elem * _numel(s) for _, s in shapes]
    offs, tot = [], 0
    for n in sizes:
        offs.append(tot)
        tot += (n + 255) // 256 * 256
    arena = torch.empty(tot, dtype=torch.uint8, device=dev)
    views = []
    for i, ((name, s), off, n) in enumerate(zip(shapes, offs, sizes)):
        v = arena[off:off + n]
        if seed_base is not None:
            ros.synth_bf16(v, seed_base + i)
        views.append((name, v))
    return arena, views


def tp_dim(name: str):
    """Megatron-style TP split of a Llama/Qwen tensor: column-parallel (dim 0)
    for q/k/v/gate/up/embed/lm_head and biases, row-parallel (dim 1) for
    o_proj/down_proj, replicated norms."""
    if "norm" in name:
        return None
    if "o_proj" in name or "down_proj" in name:
        return 1
    return 0


def tp_slice(shape, elem, dim, tp, rank):
    from paper_2604_09107_b200.ros import tp_slice as ts
    return ts(shape, elem, dim, tp, rank)


def _numel(shape):
    n = 1
    for d in shape:
        n *= d
    return n


# ------------------------------------------------------------- CPU legs
def workload_label(workload: str, receivers: int) -> str:
    """config.workload, identical in both arms for the same (workload, N)."""
    return f"{workload}: trainer -> {receivers} reader{'s' if receivers != 1 else ''}, full model"


_HOST = {}


def host_workload(shapes):
    """The workload's synthetic bytes in host memory (SURVEY.md §8d
    generator, seed 42 + i, the oracle's C restatement -- bit-identical to
    the device generator), made once per process on every host core (the C
    generator runs outside the GIL)."""
    key = tuple((n, tuple(s)) for n, s in shapes)
    if key in _HOST:
        return _HOST[key]
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from concurrent.futures import ThreadPoolExecutor

    import numpy as np

    import oracle as O
    arrs = [np.empty(_numel(s), np.uint16) for _, s in shapes]
    lib = O.port()
    step = 1 << 26  # elements per task

    def fill(job):
        i, first, n = job
        lib.ro_synth_bf16(42 + i, first, n, arrs[i][first:first + n].ctypes.data)

    jobs = [(i, f, min(step, a.size - f)) for i, a in enumerate(arrs) for f in range(0, a.size, step)]
    with ThreadPoolExecutor(os.cpu_count() or 1) as ex:
        list(ex.map(fill, jobs))
    _HOST.clear()
    _HOST[key] = [a.view(np.uint8) for a in arrs]
    return _HOST[key]


def cpu_reference_run(shapes, readers: int = 1, steps: int = 1, warmup: int = 0,
                      verify: bool = True):
    """The reference refstore (oracle/_ref, compiled from its own sources)
    pulling the WHOLE workload through its own public API and stock path:
    ClientCore publish / replicate over MemNetwork (transport_mem.cpp:170-201:
    memcpy under the source's lock + digest64 per item on the reader).
    Throughput mode (SURVEY.md §8d ii): one ThreadExecutor per replica,
    server and client pipelines off, so `readers` readers pull from the
    trainer in parallel, each on its own executor thread.  The trainer
    publishes once; every step adds `readers` fresh replicas that land the
    full model into the same host buffers, then closes them.  Returns the
    per-step results (value = bytes landed by all readers / wall time of
    the step's replicate fan-out)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import numpy as np

    import oracle as O
    if not O.ref_available():
        return None
    t0 = time.perf_counter()
    src = host_workload(shapes)
    gen_s = time.perf_counter() - t0
    total = sum(a.nbytes for a in src)
    # one landing copy per reader when the host has the memory (N=8: 8 x 16 GB);
    # otherwise the readers land into shared buffers (identical bytes), said so
    # in `sample`
    try:
        import psutil
        avail = psutil.virtual_memory().available
    except Exception:  # noqa: BLE001
        avail = None
    shared = avail is not None and readers * total > 0.85 * avail  # the source copy is already resident
    if shared:
        one = [np.empty_like(a) for a in src]
        dst = [one] * readers
    else:
        dst = [[np.empty_like(a) for a in src] for _ in range(readers)]
    c = O.RefCluster(threaded=True, server_pipeline=False, client_pipeline=False)
    c.add("trainer")
    for (name, _), a in zip(shapes, src):
        assert c.register("trainer", 0, name, a) == 0
    st, publish_s = c.publish("trainer", 1)
    assert st == 0, st
    out = []
    for k in range(warmup + steps):
        names = [f"reader{k}_{j}" for j in range(readers)]
        for nm, bufs in zip(names, dst):
            c.add(nm)
            for (name, _), b in zip(shapes, bufs):
                assert c.register(nm, 0, name, b) == 0
        sts, _, _, secs = c.pull_many(names)
        assert sts == [0] * readers, sts
        if verify and k == 0:
            for bufs in dst:
                assert all(np.array_equal(a, b) for a, b in zip(src, bufs)), "reference bytes differ"
        for nm in names:
            c.close_replica(nm)
        if k >= warmup:
            out.append(secs)
    c.close()
    sec = statistics.median(out)
    nproc = os.cpu_count() or 1
    return {"value": readers * total / sec / 1e9, "unit": UNIT, "cores": min(readers, nproc),
            "nproc": nproc, "kind": "reference", "steps_s": [round(x, 4) for x in out],
            "publish_s": round(publish_s, 3), "host_gen_s": round(gen_s, 2),
            "sample": f"whole workload ({len(shapes)} tensors, {total / 1e9:.3f} GB) per step: "
                      f"refstore publish once, then per step {readers} fresh reader replica(s) "
                      f"replicate('latest') through ClientCore + MemNetwork, ThreadExecutor per "
                      f"replica, pipeline off; copy + digest64 run on each reader's executor "
                      f"thread ({min(readers, nproc)} core(s) busy of {nproc}); median of {len(out)}"
                      + ("; host RAM short of one copy per reader: the readers share one set of "
                         "landing buffers" if shared else "")}


def reference_parity(workload, t, r, rviews, cast: bool, soft: bool = False, chunk: int = 4096):
    """Pre-timing parity against the reference at full scale
    (tests/golden/scale.json, made by tests/golden/make_scale_golden.py from
    oracle/_ref): the trainer's manifest bytes (build_publish_payload), the
    reader's chunk-digest table, and the reference digest64 of every landed
    tensor (its e4m3 cast for config 5).  None when no fixture covers it."""
    import hashlib

    import numpy as np

    from paper_2604_09107_b200 import ros
    key = {"llama3_8b": "config2_llama3_8b", "llama3_70b_tp8": "config5_llama3_70b_tp8"}.get(workload)
    path = os.path.join(ROOT, "tests", "golden", "scale.json")
    if key is None or not os.path.exists(path):
        return None
    with open(path) as f:
        g = json.load(f)[key]
    sha = lambda a: hashlib.sha256(np.ascontiguousarray(a).astype("<u8").tobytes()).hexdigest()
    landed = ros.digest_spans([w.data_ptr() for _, w in rviews], [w.numel() for _, w in rviews],
                              rviews[0][1].device.index or 0)
    want = g["cast_digests"] if cast else g["tensor_digests"]
    out = {"manifest": hashlib.sha256(t.manifest(0)).hexdigest() == g["manifest_sha256"],
           # the fixture's chunk table is over 4096-byte chunks
           "chunk_table": sha(r.chunk_digests(0)) == g["chunk_table_sha256"] if chunk == 4096 else None,
           "landed_tensors": ["%016X" % x for x in landed] == want,
           "against": "tests/golden/scale.json (reference digest64 / build_publish_payload)"}
    if not soft:
        assert out["manifest"] and out["chunk_table"] is not False and out["landed_tensors"], out
    return out


def register_pair(t, r, shapes, tviews, rviews, dev, reshard: bool, cast: bool):
    """Registers the trainer's and the reader's regions the way every bench
    mode (and tests/test_scale_parity.py) lays them out.  Plain: whole tensors
    on both sides.  cast: the reader lands each tensor as e4m3 (config 5).
    reshard: the trainer holds TP=1 tensors (one shard) or FSDP row blocks
    (t.num_shards > 1: Shard(0)), the reader the two TP=2 shards of every
    tensor, landing in its arena (shard 0 then shard 1 per tensor); returns
    {(shard, name): (buffer, bytes, geometry)} of the reader's slices."""
    import torch

    from paper_2604_09107_b200.ros import Status
    fsdp = t.num_shards
    rslices = {}
    for (n, v), (_, w), (_, shape) in zip(tviews, rviews, shapes):
        if cast:
            assert t.register_tensor(0, n, v) == Status.ok
            assert r.register_cast(0, n, w, v.numel()) == Status.ok
            continue
        if not reshard:
            assert t.register_tensor(0, n, v) == Status.ok
            assert r.register_tensor(0, n, w) == Status.ok
            continue
        for i in range(fsdp):
            g = tp_slice(shape, 2, 0 if fsdp > 1 else None, fsdp, i)
            rows, wb, r0, nr, c0, nc = g
            off = r0 * wb + c0
            assert t.register_slice(i, n, v[off:off + nr * nc], g) == Status.ok
        dim = tp_dim(n)
        for sh in range(2):
            geo = tp_slice(shape, 2, dim, 2, sh)
            off = 0 if sh == 0 else rslices[(0, n)][1]
            if dim is None and sh == 1:  # replicated: every shard holds it whole
                buf = torch.empty(geo[3] * geo[5], dtype=torch.uint8, device=dev)
            else:
                buf = w[off:off + geo[3] * geo[5]]
            rslices[(sh, n)] = (buf, geo[3] * geo[5], geo)
            assert r.register_slice(sh, n, buf, geo) == Status.ok
    return rslices


# ------------------------------------------------------------- our arm
def run_single(args):
    import torch

    from paper_2604_09107_b200.ros import Cluster, Status
    dev = torch.device("cuda:0")
    shapes = workload_shapes(args.workload)
    total = sum(2 * _numel(s) for _, s in shapes)
    log(f"[bench] workload {args.workload}: {len(shapes)} tensors, {total / 1e9:.3f} GB")
    tarena, tviews = alloc_replica(shapes, dev, seed_base=42)
    cast = args.cast
    if cast and args.reshard != "none":
        raise SystemExit("--cast is measured on the same-slicing pull (config 5)")
    rarena, rviews = alloc_replica(shapes, dev, elem=1 if cast else 2)
    torch.cuda.synchronize()
    stream = torch.cuda.Stream(device=dev)
    cl = Cluster()
    t = cl.open("m", "trainer", 8 if args.reshard == "fsdp_tp2" else 1, chunk_bytes=args.chunk,
                early_publish=args.early_publish)
    reshard = args.reshard in ("tp2", "fsdp_tp2")
    fsdp = t.num_shards  # trainer shards (FSDP-8: Shard(0) row blocks)
    r = cl.open("m", "rollout1", 2 if reshard else 1, chunk_bytes=args.chunk)
    rslices = register_pair(t, r, shapes, tviews, rviews, dev, reshard, cast)
    for s in range(r.num_shards):
        r.set_stream(s, stream)
    t0 = time.perf_counter()
    assert t.publish(1).status == Status.ok
    publish_s = time.perf_counter() - t0
    publish_ms = t.stats().last_publish_ms

    def step():
        if r.is_published:
            assert r.unpublish().status == Status.ok
        r.invalidate()
        w0 = time.perf_counter()
        res = r.replicate("latest")
        w1 = time.perf_counter()
        assert res.status == Status.ok, res
        return w1 - w0

    def verify():
        if cast:
            # against the standalone K5 kernel (itself checked against the
            # oracle on all 65536 bf16 patterns in tests/test_gpu_kernels.py)
            from paper_2604_09107_b200 import ros
            for (n, v), (_, w) in zip(tviews, rviews):
                want = torch.empty_like(w)
                ros.bf16_to_e4m3(v, want)
                torch.cuda.synchronize()
                assert torch.equal(w, want), n
            assert (r.chunk_digests(0) == t.chunk_digests(0)).all()
            return
        if not reshard:
            assert torch.equal(tarena, rarena), "reader bytes differ from trainer"
            assert (r.chunk_digests(0) == t.chunk_digests(0)).all()
            return
        for (n, v), (_, shape) in zip(tviews, shapes):
            for s in range(2):
                buf, nb, (rows, w, r0, nr, c0, nc) = rslices[(s, n)]
                want = v.view(rows, w)[r0:r0 + nr, c0:c0 + nc]
                assert torch.equal(buf.view(nr, nc), want), (s, n)

    # the first pull right after the publish: the weight-update latency a
    # reader sees from the trainer's publish call (with --early-publish the
    # big-entry digests are still running; the final manifest lands later)
    step()
    publish_to_reader_s = time.perf_counter() - t0
    assert t.finalize() == Status.ok
    publish_final_s = time.perf_counter() - t0
    for _ in range(args.warmup - 1):
        step()
    parity = None
    if not args.no_verify:
        verify()
        if not reshard:
            parity = reference_parity(args.workload, t, r, rviews, cast, chunk=args.chunk)
    clk = ClockSampler(0)
    torch.cuda.synchronize()
    clk.start()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    kernel_ms, walls, fill_ms = [], [], []
    pulled0 = r.stats().bytes_pulled
    h2d0, d2h0 = r.stats().h2d_bytes, r.stats().d2h_bytes
    launches0 = r.stats().kernel_launches
    ev0.record(stream)
    for _ in range(args.steps):
        e_a, e_b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e_a.record(stream)
        walls.append(step())
        e_b.record(stream)
        e_b.synchronize()
        # single reader shard: the pull kernel's own CUDA-event time; reshard:
        # the step's device time on the shards' stream (both shard kernels)
        kernel_ms.append(r.stats().last_pull_ms if not reshard else e_a.elapsed_time(e_b))
        fill_ms.append(r.stats().fill_sum_ms)  # the pull kernels alone (CUDA events)
    ev1.record(stream)
    torch.cuda.synchronize()
    clocks = clk.stop()
    dev_ms = ev0.elapsed_time(ev1)
    st = r.stats()
    landed = st.bytes_pulled - pulled0
    if not reshard:
        assert landed == args.steps * total, (landed, total)
    if not args.no_verify:
        verify()
    value = landed / (dev_ms / 1e3) / 1e9
    e2e = landed / sum(walls) / 1e9
    k_avg = statistics.mean(kernel_ms)
    fills_per_step = r.num_shards if reshard else 1
    fill_avg = statistics.mean(fill_ms) / fills_per_step  # one pull launch
    n_chunks = sum((2 * _numel(s) + args.chunk - 1) // args.chunk for _, s in shapes)
    # algorithmic bytes per launch: read source + write destination + read the
    # source chunk table + write own table + watermark words
    alg = (total + total // 2 if cast else 2 * total) + 16 * n_chunks + 4 * ((n_chunks + 31) // 32)
    peaks = measured_peaks()
    # reshard: the roofline is the pull kernel's (one launch per reader shard,
    # alg / shards each); the step adds the slice copies, group packing and
    # host work between launches (step_frac)
    achieved = (alg / fills_per_step) / (fill_avg / 1e3) / 1e9 if reshard else alg / (k_avg / 1e3) / 1e9
    line = {
        "metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(dev_ms / args.steps, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "config": {"workload": workload_label(args.workload, 1)
                               + (f", resharded {'FSDP-8' if fsdp > 1 else 'TP=1'} -> TP=2 "
                                  "(all shards on this GPU)" if reshard else "")
                               + (", landed as fp8 e4m3 (fused cast; bytes = bf16 ingress)" if cast else ""),
                   "placement": "trainer and reader regions in the HBM of one GPU (local pull)",
                   "bytes_per_receiver": total, "tensors": len(shapes), "chunk_bytes": args.chunk,
                   "receivers": 1, "l2": "inputs (16 GB/replica) >> 126 MB L2; no flush"},
        "per_receiver_gbs": [round(value, 2)],
        "weight_update_latency_s": round(statistics.mean(walls), 5),
        "publish_s": round(publish_s, 4), "publish_device_ms": round(publish_ms, 3),
        "publish_to_first_reader_s": round(publish_to_reader_s, 4),
        "publish_final_s": round(publish_final_s, 4), "early_publish": args.early_publish,
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peaks["hbm_gbs"],
                     "unit": "GB/s", "frac": round(achieved / peaks["hbm_gbs"], 4),
                     "traffic": ncu_traffic("reshard" if reshard else "cast" if cast else "local",
                                            workload=args.workload)
                     if args.reshard in ("none", "fsdp_tp2") else None,
                     "peak_src": peaks["src"],
                     "kernel": "pull_tma_kernel",
                     "kernel_ms_avg": round(fill_avg if reshard else k_avg, 3),
                     "alg_bytes_per_launch": alg // fills_per_step,
                     **({"step_ms": round(k_avg, 3), "launches_per_step": fills_per_step,
                         "step_frac": round(alg / (k_avg / 1e3) / 1e9 / peaks["hbm_gbs"], 4)}
                        if reshard else {})},
        "e2e": {"value": round(e2e, 2), "unit": UNIT,
                "h2d_bytes_per_step": (st.h2d_bytes - h2d0) // args.steps,
                "d2h_bytes_per_step": (st.d2h_bytes - d2h0) // args.steps,
                "what": "wall clock of rs_replicate (plan+bind+kernel+unpack+complete) per step, "
                        "version resident in the trainer's HBM"},
        "parity": parity,
        "gpu_launches": st.kernel_launches - launches0,  # the reader's kernels in the timed steps (counted by the library)
        "clocks": clocks,
    }
    version = 1
    if not (reshard or cast):
        # Version bumps with a warm reader (config 4's bump at N=1): the
        # trainer unpublishes and publishes v+1 (same bytes), in the
        # reference order and then with early publish (the big-entry digests
        # in the background), and the reader updates.  bump = publish call +
        # update call, wall clock; final_manifest = until the reference
        # manifest is committed.
        bumps = {}
        for mode, early in (("reference_order", False), ("early_publish", True)):
            t.set_early_publish(early)
            assert t.unpublish().status == Status.ok
            b0 = time.perf_counter()
            assert t.publish(version + 1).status == Status.ok
            b1 = time.perf_counter()
            res = r.update("latest")
            b2 = time.perf_counter()
            assert res.status == Status.ok and res.version == version + 1 and res.changed, res
            assert t.finalize() == Status.ok
            b3 = time.perf_counter()
            version += 1
            bumps[mode] = {"publish_s": round(b1 - b0, 5), "update_s": round(b2 - b1, 5),
                           "bump_latency_s": round(b2 - b0, 5), "final_manifest_s": round(b3 - b0, 5)}
        t.set_early_publish(args.early_publish)
        assert r.manifest(0) == t.manifest(0)
        line["bump"] = dict(bumps, what="warm reader: trainer publish(v+1) + reader update, wall clock")
    if not (reshard or cast or args.no_host_e2e):
        # End to end from HOST buffers, through the C ABI: the version is
        # parked in pinned host memory (a retention offload, the reference's
        # own host-resident copy) and every step the reader pulls it from
        # there -- host->device bytes inside the timed region, the fill's
        # status read back.  Same metric and workload as the device arm.
        line["e2e"] = host_e2e(cl, t, r, stream, total, tarena, rarena, args, version)
        line["e2e_device_resident"] = {"value": round(e2e, 2), "unit": UNIT,
                                       "what": "rs_replicate wall clock, version in the trainer's HBM"}
    if not args.no_cpu:
        cb = cpu_reference_run(shapes, readers=1, steps=args.cpu_reps, warmup=1, verify=False)  # the warm-up takes the landing buffers' first-touch page faults
        line["cpu_baseline"] = cb and {k: cb[k] for k in ("value", "unit", "cores", "nproc", "kind",
                                                          "sample")}
    print(json.dumps(line), flush=True)
    cl.close()


def host_e2e(cl, t, r, stream, total, tarena, rarena, args, version: int = 1):
    import torch

    from paper_2604_09107_b200.ros import Status
    dev = tarena.device
    w = cl.open("m", "watcher", 1)
    wt = torch.zeros(4096, dtype=torch.uint8, device=dev)
    assert w.register_tensor(0, "w0", wt) == Status.ok
    w.set_retention([0])
    assert w.connect() == Status.ok
    if r.is_published:
        assert r.unpublish().status == Status.ok
    r.invalidate()
    assert t.unpublish().status == Status.ok  # parks v1 in pinned host memory
    assert t.lanes() == [version]
    walls = []
    h2d0, d2h0 = r.stats().h2d_bytes, r.stats().d2h_bytes
    for k in range(args.warmup + args.steps):
        if r.is_published:
            assert r.unpublish().status == Status.ok
        r.invalidate()
        torch.cuda.synchronize()
        w0 = time.perf_counter()
        res = r.replicate(str(version))
        torch.cuda.synchronize()
        if k >= args.warmup:
            walls.append(time.perf_counter() - w0)
        assert res.status == Status.ok, res
        if k == 0:
            h2d0, d2h0 = r.stats().h2d_bytes, r.stats().d2h_bytes
            srcs = {a.src for a in cl.assigns() if a.replica == r.replica}
            assert f"trainer+offload@{version}" in srcs, srcs
    if not args.no_verify:
        assert torch.equal(tarena, rarena), "bytes pulled from the host offload differ"
    st = r.stats()
    steps = args.warmup + args.steps - 1
    return {"value": round(total / statistics.mean(walls) / 1e9, 2), "unit": UNIT,
            "h2d_bytes_per_step": total + (st.h2d_bytes - h2d0) // max(steps, 1),
            "d2h_bytes_per_step": (st.d2h_bytes - d2h0) // max(steps, 1),
            "what": "rs_replicate wall clock per step with the version in pinned HOST memory "
                    "(a retention offload): every byte crosses host->device inside the timed "
                    "region (PCIe: copy-engine frames into the landing regions, verified in place "
                    "by the pull kernel); status read back"}


def run_reference(args):
    """--impl reference: the reference's own CPU implementation of the path
    (oracle/_ref), same workload, metric and config.workload as our arm at
    this N: rank 0 alone runs it with N-1 readers (1 at N=1)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    readers = max(1, max(world, args.gpus) - 1)
    shapes = workload_shapes(args.workload)
    r = cpu_reference_run(shapes, readers=readers, steps=args.steps, warmup=args.warmup,
                          verify=not args.no_verify)
    if r is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built"}))
        return
    v = r["value"]
    total = sum(2 * _numel(s) for _, s in shapes)
    line = {"impl": "reference", "metric": METRIC, "value": round(v, 3), "unit": UNIT,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(1e3 * statistics.median(r["steps_s"]), 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64",
            "data": "synthetic",
            "config": {"workload": workload_label(args.workload, readers),
                       "placement": "host DRAM (the reference is a CPU library)",
                       "bytes_per_receiver": total, "tensors": len(shapes), "receivers": readers},
            "cpu_baseline": {"value": round(v, 3), "unit": UNIT, "cores": r["cores"],
                             "nproc": r["nproc"], "kind": "reference", "sample": r["sample"]},
            "publish_s": r["publish_s"],
            "e2e": {"value": round(v, 3), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="llama3_8b")
    ap.add_argument("--chunk", type=int, default=4096)
    ap.add_argument("--no-verify", action="store_true")
    ap.add_argument("--fanout", default="chain", choices=["chain", "pairs", "ring"])
    ap.add_argument("--reshard", default="none", choices=["none", "tp2", "fsdp_tp2"])
    ap.add_argument("--cast", action="store_true", help="reader lands fp8 e4m3 (config 5)")
    ap.add_argument("--scenario", default="steady", choices=["steady", "elastic"],
                    help="elastic: config 4 (join at 50%% + version bump), N >= 3")
    ap.add_argument("--early-publish", action="store_true",
                    help="trainer publishes early: chunk table + manifest structure first, "
                         "big-entry digests in the background (rs_config.early_publish)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-host-e2e", action="store_true",
                    help="skip the host-buffer end-to-end leg (N=1)")
    ap.add_argument("--cpu-reps", type=int, default=2,
                    help="cpu_baseline: whole-workload reference pulls timed in our arm's line")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1 or args.gpus > 1:
        from paper_2604_09107_b200 import bench_dist
        return bench_dist.run(args)
    return run_single(args)


if __name__ == "__main__":
    main()
