"""N-GPU leg of bench.py (torchrun, one rank per GPU).

Rank 0 publishes the workload (trainer); ranks 1..N-1 are readers.  Each step
every reader drops its copy and replicates "latest"; the replicated registry
plans a chain (trainer -> r1 -> ... -> r{N-1}, the reference planner's order
for simultaneous readers) and every reader's pull kernel chases its
upstream's device watermark over NVLink (CUDA IPC peer mappings).  Per-step
device time = max over ranks of the reader kernels' CUDA-event time; `value`
= bytes landed by all readers / that time.
"""
from __future__ import annotations

import json
import os
import statistics
import sys
import time


def run(args):
    if getattr(args, "scenario", "steady") == "elastic":
        return run_elastic(args)
    if getattr(args, "reshard", "none") == "fsdp_tp2":
        return run_fsdp_tp2(args)
    if getattr(args, "reshard", "none") == "tp2":
        return run_tp2_fanout(args)
    if getattr(args, "fanout", "chain") == "ring":
        return run_ring(args)
    import torch
    import torch.distributed as dist

    import bench as B
    from paper_2604_09107_b200 import ros
    from paper_2604_09107_b200.dist import DistCluster
    from paper_2604_09107_b200.ros import Status

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    if world < 2:
        raise SystemExit("--gpus N>1 must be launched with torchrun (one rank per GPU)")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("gloo")
    dc = DistCluster()
    # the planner's topology term from the box's NVLink state (NVML); every
    # pair of an NVSwitch box is one hop, so the plan stays the reference's
    topo = ros.nvlink_cost_matrix(world) if rank == 0 else None
    dc.set_topology([f"rank{i}:cuda{i}" for i in range(world)], topo or [])
    shapes = B.workload_shapes(args.workload)
    total = sum(2 * B._numel(s) for _, s in shapes)
    # chain (default): rank 0 trains, ranks 1.. read (planner: a chain).
    # pairs: even ranks train, odd ranks read (diagnostic: no GPU both
    # sends and receives).
    pairs = getattr(args, "fanout", "chain") == "pairs"
    is_trainer = rank % 2 == 0 if pairs else rank == 0
    arena, views = B.alloc_replica(shapes, dev, seed_base=42 if is_trainer else None)
    torch.cuda.synchronize()
    name = (f"trainer{rank}" if pairs else "trainer") if is_trainer else f"rollout{rank}"
    h = dc.create("m", name, 1, chunk_bytes=args.chunk, pull_timeout_s=30.0)
    for n, v in views:
        assert h.register_tensor(0, n, v) == Status.ok
    dc.open(h, endpoints=[f"rank{rank}:cuda{local}"])
    stream = torch.cuda.Stream(device=dev)
    h.set_stream(0, stream)
    t0 = time.perf_counter()
    r = None
    for tr in ([x for x in range(world) if x % 2 == 0] if pairs else [0]):
        rr = dc.publish(h if rank == tr else None, 1)
        if rank == tr:
            r = rr
    publish_s = time.perf_counter() - t0
    if is_trainer:
        assert r.status == Status.ok, r
    reader = None if is_trainer else h

    def step():
        dc.unpublish(reader if (reader is not None and reader.is_published) else None)
        if reader is not None:
            reader.invalidate()
        dist.barrier(group=dc.pg)
        torch.cuda.synchronize()
        w0 = time.perf_counter()
        res = dc.replicate(reader, "latest")
        torch.cuda.synchronize()
        wall = time.perf_counter() - w0
        if reader is not None:
            assert res.status == Status.ok, res
            return wall, reader.stats().last_pull_ms, reader.stats().last_pull_bytes
        return wall, 0.0, 0

    for _ in range(args.warmup):
        step()

    def table_hash():
        import hashlib
        return hashlib.sha256(h.chunk_digests(0).tobytes()).hexdigest()

    # every reader's chunk-digest table (computed from the bytes it landed)
    # must equal the trainer's (computed at publish from the source bytes)
    hashes = dc.gather(None if args.no_verify else table_hash())
    verified = args.no_verify or all(x == hashes[0] for x in hashes)
    # every rank (trainer and readers) against the reference at full scale
    # (tests/golden/scale.json): manifest bytes, chunk table, landed tensors
    parity = dc.gather(None if args.no_verify else
                       B.reference_parity(args.workload, h, h, views, False, soft=True, chunk=args.chunk))
    clk = B.ClockSampler(local)
    nvc = B.NvlinkCounters(local)
    dist.barrier(group=dc.pg)
    torch.cuda.synchronize()
    clk.start()
    link0 = nvc.read()
    kl0 = h.stats().kernel_launches
    walls, kms, landed = [], [], 0
    for _ in range(args.steps):
        w, k, b = step()
        walls.append(w)
        kms.append(k)
        landed += b
    torch.cuda.synchronize()
    link1 = nvc.read()
    kl1 = h.stats().kernel_launches
    clocks = clk.stop()
    # max over ranks of per-step device time; sum of landed bytes
    t = torch.tensor([max(kms) if kms else 0.0, sum(kms), float(landed), max(walls), sum(walls)],
                     dtype=torch.float64)
    allv = [None] * world
    dist.all_gather_object(allv, (t.tolist(), kms, clocks, link0, link1, kl1 - kl0), group=dc.pg)
    step_dev_ms = [max(a[1][i] for a in allv) for i in range(args.steps)]
    total_landed = sum(a[0][2] for a in allv)
    dev_s = sum(step_dev_ms) / 1e3
    wall_s = max(a[0][4] for a in allv)
    receivers = world // 2 if pairs else world - 1
    assert total_landed == args.steps * receivers * total, (total_landed, total)
    hashes = dc.gather(None if args.no_verify else table_hash())
    verified = verified and (args.no_verify or all(x == hashes[0] for x in hashes))
    host_e2e = None
    plan = [f"{a.replica}<-{a.src}" for a in dc.assigns()][-receivers:]
    if not pairs and not getattr(args, "no_host_e2e", False):
        host_e2e = _dist_host_e2e(dc, h, reader, rank, dev, total, receivers, args)
    if rank == 0:
        per_rx = [round(total / (statistics.mean(a[1]) / 1e3) / 1e9, 2) for a in allv
                  if a[1] and statistics.mean(a[1]) > 0]
        value = total_landed / dev_s / 1e9
        mean_rx = statistics.mean(per_rx)
        line = {
            "metric": B.METRIC, "value": round(value, 2), "unit": B.UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(sum(step_dev_ms) / args.steps, 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
            "config": {"workload": B.workload_label(args.workload, receivers),
                       "placement": "trainer on GPU0, reader i on GPU i: chained fan-out over NVLink",
                       "bytes_per_receiver": total,
                       "receivers": receivers, "chunk_bytes": args.chunk,
                       "plan": plan,
                       "l2": "inputs (16 GB/replica) >> 126 MB L2; no flush"},
            "per_receiver_gbs": per_rx,
            "weight_update_latency_s": round(wall_s / args.steps, 5),
            "publish_s": round(publish_s, 4),
            "roofline": {"bound": "nvlink", "achieved": round(mean_rx, 1), "peak": 900.0,
                         "unit": "GB/s", "frac": round(mean_rx / 900.0, 4),
                         "traffic": B.ncu_traffic("nvlink", total),
                         "traffic_src": "NVLink bytes received per launch (user + read-response protocol), "
                                        "ncu nvlrx ratio from profiles/r1/ncu_nvlink_counters.json",
                         "peak_src": "nominal NVLink5 per direction "
                         "(measured peer copy 777 GB/s)", "kernel": "pull_tma_kernel",
                         "kernel_ms_avg": round(statistics.mean(step_dev_ms), 3),
                         "alg_bytes_per_launch": total,
                         # link-level accounting from ncu nvlrx/nvltx counters
                         # (profiles/r1/ncu_nvlink_counters.json): read
                         # responses carry 12.5% protocol, read requests 18.75%
                         # of the data in the other direction
                         "protocol_peak_per_receiver": [
                             round(B.NVL_ONE_WAY if i == receivers - 1 else B.NVL_BOTH_WAYS, 1)
                             for i in range(receivers)],
                         "protocol_frac": round(statistics.mean(
                             x / (B.NVL_ONE_WAY if i == len(per_rx) - 1 else B.NVL_BOTH_WAYS)
                             for i, x in enumerate(per_rx)), 4)},
            "e2e": {"value": round(total_landed / wall_s / 1e9, 2), "unit": B.UNIT,
                    "h2d_bytes_per_step": None, "d2h_bytes_per_step": None,
                    "what": "wall clock of the collective replicate (plan+bind+IPC exchange+kernel), "
                            "version resident in the trainer's HBM"},
            "gpu_launches": sum(a[5] for a in allv),  # every rank's kernels in the timed steps
            "parity": {"per_rank": parity,
                       "all": all(p and p["manifest"] and p["chunk_table"] and p["landed_tensors"]
                                  for p in parity) if not args.no_verify and parity[0] else None},
            "clocks": allv[0][2] if allv[0][2].get("sm_mhz") else allv[1][2],
            "verified": verified,
        }
        # NVML link counters over the timed steps: raw bytes (data + protocol)
        # each GPU's port sent and received, per step, and as a rate over the
        # steps' pull-kernel time against the 900 GB/s per direction
        kern_s = sum(step_dev_ms) / 1e3
        links = []
        for r, a in enumerate(allv):
            l0, l1 = a[3], a[4]
            if not (l0 and l1):
                links.append({"rank": r, "counters": None})
                continue
            tx, rx = (l1[0] - l0[0]) / args.steps, (l1[1] - l0[1]) / args.steps
            links.append({"rank": r, "tx_gb_per_step": round(tx / 1e9, 3), "rx_gb_per_step": round(rx / 1e9, 3),
                          "tx_frac_900": round(tx * args.steps / kern_s / 900e9, 4),
                          "rx_frac_900": round(rx * args.steps / kern_s / 900e9, 4)})
        line["nvlink_counters"] = {"per_rank": links, "source": next((a[4][2] for a in allv if a[4]), None),
                                   "denominator": "sum of the steps' pull-kernel time (max over readers)"}
        if host_e2e is not None:
            line["e2e_device_resident"] = line["e2e"]
            line["e2e"] = host_e2e
        # cpu_baseline: rank 0 at N=1 only (bench.py); at this N the reference
        # arm (--impl reference) times the same workload with N-1 readers
        print(json.dumps(line), flush=True)
    dist.barrier(group=dc.pg)
    dc.close()
    dist.destroy_process_group()


def _dist_host_e2e(dc, h, reader, rank, dev, total, receivers, args):
    """End to end from HOST buffers at N GPUs: the trainer's version is parked
    in pinned host memory (a retention offload on GPU0's host) and the
    readers replicate it: the first pulls it host->device over PCIe, the rest
    chase along the NVLink chain.  Wall clock per step, max over ranks."""
    import torch
    import torch.distributed as dist

    from paper_2604_09107_b200.ros import Status
    w = None
    if rank == 0:
        w = dc.create("m", "watcher", 1)
        assert w.register_tensor(0, "w0", torch.zeros(4096, dtype=torch.uint8, device=dev)) == 0
        w.set_retention([0])
    dc.open(w)
    dc.unpublish(reader if (reader is not None and reader.is_published) else None)
    r = dc.unpublish(h if rank == 0 else None)  # the last durable copy: parked in host memory
    if rank == 0:
        assert r.status == Status.ok and h.lanes() == [1], (r, h.lanes())
    walls = []
    h2d0 = d2h0 = 0
    for k in range(args.warmup + args.steps):
        dc.unpublish(reader if (reader is not None and reader.is_published) else None)
        if reader is not None:
            reader.invalidate()
        dist.barrier(group=dc.pg)
        torch.cuda.synchronize()
        w0 = time.perf_counter()
        res = dc.replicate(reader, "1")
        torch.cuda.synchronize()
        if k >= args.warmup:
            walls.append(time.perf_counter() - w0)
        if reader is not None:
            assert res.status == Status.ok, res
            if k == args.warmup - 1 or (args.warmup == 0 and k == 0):
                h2d0, d2h0 = reader.stats().h2d_bytes, reader.stats().d2h_bytes
    st = reader.stats() if reader is not None else None
    src = {a.replica: a.src for a in dc.assigns() if a.version == 1}
    per = dc.gather((sum(walls), None if st is None else (st.h2d_bytes - h2d0, st.d2h_bytes - d2h0)))
    wall = max(p[0] for p in per) / max(len(walls), 1)
    h2d = sum(p[1][0] for p in per if p[1]) // max(len(walls), 1)
    d2h = sum(p[1][1] for p in per if p[1]) // max(len(walls), 1)
    return {"value": round(receivers * total / wall / 1e9, 2), "unit": "GB/s",
            "h2d_bytes_per_step": total + h2d, "d2h_bytes_per_step": d2h,
            "first_source": src.get("rollout1"),
            "what": "collective replicate wall clock per step with the version in pinned HOST "
                    "memory (a retention offload): it crosses host->device (PCIe) inside the "
                    "timed region into the first reader, the others chase it over NVLink; "
                    "statuses read back; whole-job bytes / max-over-ranks time"}


def run_ring(args):
    """Config 5 shape: a TP-N trainer group (shard i on GPU i) pulled
    shard-for-shard by a reader group placed on GPU (i+1) mod N, optionally
    landing fp8 e4m3 (--cast).  Every GPU sends its trainer shard and
    receives its reader shard at the same time.  Both groups are replicas
    split across processes (one process per GPU holds one shard of each)."""
    import hashlib

    import torch
    import torch.distributed as dist

    import bench as B
    from paper_2604_09107_b200 import ros
    from paper_2604_09107_b200.dist import DistCluster
    from paper_2604_09107_b200.ros import Status

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("gloo")
    dc = DistCluster()
    shapes = B.workload_shapes(args.workload)
    total = sum(2 * B._numel(s) for _, s in shapes)
    cast = getattr(args, "cast", False)
    up = (rank - 1) % world  # the trainer shard this GPU's reader pulls
    tarena, tviews = B.alloc_replica(shapes, dev, seed_base=42 + 1000 * rank)
    rarena, rviews = B.alloc_replica(shapes, dev, elem=1 if cast else 2)
    torch.cuda.synchronize()
    t = dc.create("m", "trainer", world, chunk_bytes=args.chunk, pull_timeout_s=30.0)
    r = dc.create("m", "reader", world, chunk_bytes=args.chunk, pull_timeout_s=30.0)
    for (n, v), (_, w) in zip(tviews, rviews):
        assert t.register_tensor(rank, n, v) == Status.ok
        if cast:
            assert r.register_cast(up, n, w, v.numel()) == Status.ok
        else:
            assert r.register_tensor(up, n, w) == Status.ok
    dc.open(t, endpoints=[f"rank{rank}:cuda{local}"])
    dc.open(r, endpoints=[f"rank{rank}:cuda{local}"])
    stream = torch.cuda.Stream(device=dev)
    r.set_stream(up, stream)
    t0 = time.perf_counter()
    assert dc.publish(t, 1).status == Status.ok
    publish_s = time.perf_counter() - t0

    def step():
        dc.unpublish(r if r.is_published else None)
        r.invalidate()
        dist.barrier(group=dc.pg)
        torch.cuda.synchronize()
        w0 = time.perf_counter()
        res = dc.replicate(r, "latest")
        torch.cuda.synchronize()
        wall = time.perf_counter() - w0
        assert res.status == Status.ok, res
        st = r.stats()
        return wall, st.last_pull_ms, st.last_pull_bytes

    for _ in range(args.warmup):
        step()
    verified = True
    if not args.no_verify:
        # digest tables: the reader's (bf16 bytes it verified) == its trainer's
        th = hashlib.sha256(t.chunk_digests(rank).tobytes()).hexdigest()
        rh = hashlib.sha256(r.chunk_digests(up).tobytes()).hexdigest()
        allh = dc.gather((th, rh))
        verified = allh[rank][1] == allh[up][0]
        # landed bytes: regenerate the upstream shard here (same seeds) and
        # compare with the standalone K5 kernel's cast / the raw bytes
        ua, uviews = B.alloc_replica(shapes, dev, seed_base=42 + 1000 * up)
        for (n, u), (_, w) in zip(uviews, rviews):
            if cast:
                want = torch.empty_like(w)
                ros.bf16_to_e4m3(u, want)
            else:
                want = u
            torch.cuda.synchronize()
            verified &= bool(torch.equal(w, want))
        del ua, uviews
        torch.cuda.empty_cache()
        verified = all(dc.gather(verified))
    clk = B.ClockSampler(local)
    dist.barrier(group=dc.pg)
    torch.cuda.synchronize()
    clk.start()
    kl0 = r.stats().kernel_launches
    walls, kms, landed = [], [], 0
    for _ in range(args.steps):
        w, k, b = step()
        walls.append(w)
        kms.append(k)
        landed += b
    clocks = clk.stop()
    kl = r.stats().kernel_launches - kl0
    allv = dc.gather((kms, landed, sum(walls), clocks, kl))
    step_dev_ms = [max(a[0][i] for a in allv) for i in range(args.steps)]
    total_landed = sum(a[1] for a in allv)
    assert total_landed == args.steps * world * total, (total_landed, total)
    dev_s = sum(step_dev_ms) / 1e3
    wall_s = max(a[2] for a in allv)
    if rank == 0:
        per_rx = [round(total / (statistics.mean(a[0]) / 1e3) / 1e9, 2) for a in allv]
        mean_rx = statistics.mean(per_rx)
        line = {
            "metric": B.METRIC, "value": round(total_landed / dev_s / 1e9, 2), "unit": B.UNIT,
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(sum(step_dev_ms) / args.steps, 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
            "config": {"workload": f"{args.workload}: TP-{world} trainer shard i (GPU i) -> reader "
                                   f"shard i on GPU (i+1) mod {world}"
                                   + (", landed as fp8 e4m3 (fused cast)" if cast else ""),
                       "bytes_per_receiver": total, "receivers": world, "chunk_bytes": args.chunk,
                       "l2": "inputs >> 126 MB L2; no flush"},
            "per_receiver_gbs": per_rx,
            "weight_update_latency_s": round(wall_s / args.steps, 5),
            "publish_s": round(publish_s, 4),
            "roofline": {"bound": "nvlink", "achieved": round(mean_rx, 1), "peak": 900.0,
                         "unit": "GB/s", "frac": round(mean_rx / 900.0, 4),
                         "traffic": B.ncu_traffic("nvlink", total),
                         "traffic_src": "NVLink bytes received per launch (user + read-response protocol), "
                                        "ncu nvlrx ratio from profiles/r1/ncu_nvlink_counters.json",
                         "peak_src": "nominal NVLink5 per direction", "kernel": "pull_tma_kernel",
                         "kernel_ms_avg": round(statistics.mean(step_dev_ms), 3),
                         "alg_bytes_per_launch": total,
                         # every GPU of the ring sends and receives: read
                         # responses + the requests of the pull out of it
                         "protocol_peak": round(B.NVL_BOTH_WAYS, 1),
                         "protocol_frac": round(mean_rx / B.NVL_BOTH_WAYS, 4)},
            "e2e": {"value": round(total_landed / wall_s / 1e9, 2), "unit": B.UNIT,
                    "h2d_bytes_per_step": None, "d2h_bytes_per_step": None,
                    "what": "wall clock of the collective replicate (plan+bind+IPC exchange+kernel)"},
            "gpu_launches": sum(a[4] for a in allv),  # counted by the library
            "clocks": clocks,
            "verified": verified,
        }
        print(json.dumps(line), flush=True)
    dist.barrier(group=dc.pg)
    dc.close()
    dist.destroy_process_group()


def _synth_full(shape, seed, dev):
    import torch

    from paper_2604_09107_b200 import ros
    n = 1
    for d in shape:
        n *= d
    t = torch.empty(2 * n, dtype=torch.uint8, device=dev)
    ros.synth_bf16(t, seed)
    return t


def _piece(full, geo):
    rows, w, r0, nr, c0, nc = geo
    return full.view(rows, w)[r0:r0 + nr, c0:c0 + nc].contiguous().view(-1)


def run_fsdp_tp2(args):
    """Config 3: a trainer sharded FSDP-N (Shard(0): shard i = rows
    [i*R/N, (i+1)*R/N) of every tensor, on GPU i) is pulled by N/2 rollout
    replicas in the TP-2 layout (column-parallel q/k/v/gate/up/embed/lm_head
    and biases, row-parallel o/down, replicated norms); replica j's shard s
    lives on GPU 2j+s.  All replicas replicate at once: the planner has
    replica 0 reshard from the N FSDP sources and chains the others onto the
    same-slicing copy before them, each chasing its upstream's watermarks.
    Both groups are replicas split across processes (one process per GPU)."""
    import hashlib

    import torch
    import torch.distributed as dist

    import bench as B
    from paper_2604_09107_b200.dist import DistCluster
    from paper_2604_09107_b200.ros import Status, tp_slice

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    if world % 2:
        raise SystemExit("--reshard fsdp_tp2 needs an even number of GPUs")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("gloo")
    dc = DistCluster()
    shapes = B.workload_shapes(args.workload)
    rep, s = rank // 2, rank % 2  # this GPU's rollout replica and TP shard
    fsdp = [tp_slice(shape, 2, 0, world, rank) for _, shape in shapes]
    tp2 = [tp_slice(shape, 2, B.tp_dim(n), 2, s) for n, shape in shapes]
    tsizes = [g[3] * g[5] for g in fsdp]
    rsizes = [g[3] * g[5] for g in tp2]

    def arena(sizes):
        offs, tot = [], 0
        for n in sizes:
            offs.append(tot)
            tot += (n + 255) // 256 * 256
        a = torch.zeros(tot, dtype=torch.uint8, device=dev)
        return a, [a[o:o + n] for o, n in zip(offs, sizes)]

    tarena, tviews = arena(tsizes)
    for i, ((n, shape), g) in enumerate(zip(shapes, fsdp)):
        full = _synth_full(shape, 42 + i, dev)
        tviews[i].copy_(_piece(full, g))
        del full
    rarena, rviews = arena(rsizes)
    torch.cuda.synchronize()
    t = dc.create("m", "trainer", world, chunk_bytes=args.chunk, pull_timeout_s=60.0)
    for (n, _), v, g in zip(shapes, tviews, fsdp):
        assert t.register_slice(rank, n, v, g) == Status.ok
    r = dc.create("m", f"tp2_{rep}", 2, chunk_bytes=args.chunk, pull_timeout_s=60.0)
    for (n, _), v, g in zip(shapes, rviews, tp2):
        assert r.register_slice(s, n, v, g) == Status.ok
    dc.open(t, endpoints=[f"rank{rank}:cuda{local}"])
    dc.open(r, endpoints=[f"rank{rank}:cuda{local}"])
    stream = torch.cuda.Stream(device=dev)
    r.set_stream(s, stream)
    t0 = time.perf_counter()
    assert dc.publish(t, 1).status == Status.ok
    publish_s = time.perf_counter() - t0

    def step():
        dc.unpublish(r if r.is_published else None)
        r.invalidate()
        dist.barrier(group=dc.pg)
        torch.cuda.synchronize()
        w0 = time.perf_counter()
        res = dc.replicate(r, "latest")
        torch.cuda.synchronize()
        wall = time.perf_counter() - w0
        assert res.status == Status.ok, res
        st = r.stats()
        return wall, st.last_pull_ms, st.last_pull_bytes

    for _ in range(args.warmup):
        step()
    verified = True
    if not args.no_verify:
        # the landed TP-2 slices against slices of the regenerated tensors
        for i, ((n, shape), g) in enumerate(zip(shapes, tp2)):
            full = _synth_full(shape, 42 + i, dev)
            verified &= bool(torch.equal(rviews[i], _piece(full, g)))
            del full
        # same-slicing replicas hold identical chunk-digest tables
        hs = dc.gather((s, hashlib.sha256(r.chunk_digests(s).tobytes()).hexdigest()))
        for sh in (0, 1):
            verified &= len({h for x, h in hs if x == sh}) == 1
        verified = all(dc.gather(verified))
    clk = B.ClockSampler(local)
    dist.barrier(group=dc.pg)
    torch.cuda.synchronize()
    clk.start()
    kl0 = (r.stats().kernel_launches if r is not None else 0)
    walls, kms, landed = [], [], 0
    for _ in range(args.steps):
        w, k, b = step()
        walls.append(w)
        kms.append(k)
        landed += b
    clocks = clk.stop()
    kl = (r.stats().kernel_launches if r is not None else 0) - kl0
    kls = dc.gather(kl)  # collective: every rank
    # Roofline of this shard's fill: bytes that cross NVLink (from sources on
    # other GPUs) vs bytes read from local HBM, all written to local HBM.
    src = {a.replica: a.src for a in dc.assigns()}.get(f"tp2_{rep}")
    remote = local_b = 0
    from_gpu = {}  # source GPU -> bytes this shard pulls from it
    for (n, shape), g in zip(shapes, tp2):
        if src != "trainer":  # a same-slicing upstream replica: shard s on GPU 2*up + s
            up = int(src.split("_")[1])
            from_gpu[2 * up + s] = from_gpu.get(2 * up + s, 0) + g[3] * g[5]
            remote += g[3] * g[5]
            continue
        for i in range(world):
            fg = tp_slice(shape, 2, 0, world, i)
            a0, a1 = max(g[2], fg[2]), min(g[2] + g[3], fg[2] + fg[3])
            c0, c1 = max(g[4], fg[4]), min(g[4] + g[5], fg[4] + fg[5])
            if a0 < a1 and c0 < c1:
                from_gpu[i] = from_gpu.get(i, 0) + (a1 - a0) * (c1 - c0)
                if i == rank:
                    local_b += (a1 - a0) * (c1 - c0)
                else:
                    remote += (a1 - a0) * (c1 - c0)
    hbm = B.measured_peaks()["hbm_gbs"] * 1e9
    t_min = max(remote / 900e9, (local_b + sum(rsizes)) / hbm)
    allv = dc.gather((kms, landed, sum(walls), clocks, sum(rsizes), rep, s, remote, local_b, t_min,
                      from_gpu))
    step_dev_ms = [max(a[0][i] for a in allv) for i in range(args.steps)]
    total_landed = args.steps * sum(a[4] for a in allv)  # reader-layout bytes landed
    dev_s = sum(step_dev_ms) / 1e3
    wall_s = max(a[2] for a in allv)
    if rank == 0:
        per_rx = [round(a[4] / (statistics.mean(a[0]) / 1e3) / 1e9, 2) for a in allv]
        mean_rx = statistics.mean(per_rx)
        plan = sorted({f"{a.replica}<-{a.src}" for a in dc.assigns()})
        # Whole-box bound: every GPU's NVLink port and its HBM (landed writes
        # + local reads + reads served to peers); the step can be no shorter
        # than the busiest resource of the busiest GPU.  Link bytes count the
        # read-response protocol (12.5%, profiles/r1/ncu_nvlink_counters.json);
        # the read requests flowing the other way (18.75% of the data for
        # 128-byte reads, less for promoted 256-byte reads) are left out, so
        # this stays a lower bound on the step; with them: t_gpu_req.
        tx, rx, hb = [0] * world, [0] * world, [0] * world
        for g_rx, a in enumerate(allv):
            hb[g_rx] += a[4]
            for g_src, nb in a[10].items():
                hb[g_src] += nb
                if g_src != g_rx:
                    tx[g_src] += nb
                    rx[g_rx] += nb
        t_gpu = [max(max(tx[g], rx[g]) * (1 + B.NVL_RESP) / 900e9, hb[g] / hbm) for g in range(world)]
        t_gpu_req = [max((tx[g] * (1 + B.NVL_RESP) + rx[g] * B.NVL_REQ) / 900e9,
                         (rx[g] * (1 + B.NVL_RESP) + tx[g] * B.NVL_REQ) / 900e9,
                         hb[g] / hbm) for g in range(world)]
        t_box = max(t_gpu)
        line = {
            "metric": B.METRIC, "value": round(total_landed / dev_s / 1e9, 2), "unit": B.UNIT,
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(sum(step_dev_ms) / args.steps, 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
            "config": {"workload": f"{args.workload}: FSDP-{world} trainer (Shard(0), GPU i) -> "
                                   f"{world // 2} TP-2 rollout replicas (replica j on GPUs 2j, 2j+1), "
                                   "resharded on pull",
                       "bytes_per_receiver_shard": [a[4] for a in allv],
                       "receivers": world, "chunk_bytes": args.chunk, "plan": plan,
                       "l2": "inputs >> 126 MB L2; no flush"},
            "per_receiver_gbs": per_rx,
            "weight_update_latency_s": round(wall_s / args.steps, 5),
            "publish_s": round(publish_s, 4),
            "roofline": {"bound": "nvlink+hbm", "achieved": round(mean_rx, 1),
                         "peak": round(statistics.mean(a[4] for a in allv) / t_box / 1e9, 1),
                         "unit": "GB/s",
                         "frac": round(t_box / (statistics.mean(step_dev_ms) / 1e3), 4),
                         "traffic": None,
                         "peak_src": "whole box: per GPU max(NVLink tx or rx data x 1.125 read-response "
                                     "protocol / 900 GB/s per direction, HBM bytes / measured HBM peak); "
                                     "frac = busiest GPU's bound / step time",
                         "bound_ms_per_gpu": [round(t * 1e3, 3) for t in t_gpu],
                         "bound_ms_per_gpu_with_requests": [round(t * 1e3, 3) for t in t_gpu_req],
                         "nvlink_tx_bytes_per_gpu": tx, "nvlink_rx_bytes_per_gpu": rx,
                         "hbm_bytes_per_gpu": hb,
                         "frac_per_shard_naive": round(max(a[9] for a in allv) /
                                                       (statistics.mean(step_dev_ms) / 1e3), 4),
                         "nvlink_bytes_per_shard": [a[7] for a in allv],
                         "local_read_bytes_per_shard": [a[8] for a in allv],
                         "kernel": "pull_tma_kernel",
                         "kernel_ms_avg": round(statistics.mean(step_dev_ms), 3),
                         "alg_bytes_per_launch": max(a[4] for a in allv)},
            "e2e": {"value": round(total_landed / wall_s / 1e9, 2), "unit": B.UNIT,
                    "h2d_bytes_per_step": None, "d2h_bytes_per_step": None,
                    "what": "wall clock of the collective replicate (plan+bind+IPC exchange+kernel)"},
            "gpu_launches": sum(kls),  # counted by the library
            "clocks": clocks,
            "verified": verified,
        }
        print(json.dumps(line), flush=True)
    dist.barrier(group=dc.pg)
    dc.close()
    dist.destroy_process_group()


def run_elastic(args):
    """Config 4: elastic join + version bump.  Rank 0 trains; ranks
    1..N-2 replicate version v at once (a chain); rank N-1 joins when rank 1
    has verified half of its batches and is planned onto a partially landed
    copy, chasing its watermarks.  Then the trainer unpublishes v, mutates its
    weights in place (new bytes), publishes v+1 and every reader updates to
    "latest"; v copies are never v+1 sources.  Per step: the joiner's
    join -> complete latency and the bump latency (trainer unpublish ->
    every reader on v+1), max over ranks, wall clock."""
    import hashlib

    import torch
    import torch.distributed as dist

    import bench as B
    from paper_2604_09107_b200 import ros
    from paper_2604_09107_b200.dist import DistCluster
    from paper_2604_09107_b200.ros import Status

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    if world < 3:
        raise SystemExit("--scenario elastic needs >= 3 GPUs (trainer, readers, a joiner)")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("gloo")
    dc = DistCluster()
    shapes = B.workload_shapes(args.workload)
    total = sum(2 * B._numel(s) for _, s in shapes)
    is_trainer, joiner = rank == 0, world - 1
    arena, views = B.alloc_replica(shapes, dev, seed_base=42 if is_trainer else None)
    torch.cuda.synchronize()
    name = "trainer" if is_trainer else (f"rollout{rank}" if rank != joiner else "joiner")
    early = getattr(args, "early_publish", False)
    h = dc.create("m", name, 1, chunk_bytes=args.chunk, pull_timeout_s=60.0,
                  early_publish=early and is_trainer)
    for n, v in views:
        assert h.register_tensor(0, n, v) == Status.ok
    dc.open(h, endpoints=[f"rank{rank}:cuda{local}"])
    version = 1
    dc.publish(h if is_trainer else None, version)
    reader = None if is_trainer else h

    def table():
        return hashlib.sha256(h.chunk_digests(0).tobytes()).hexdigest()

    joins, bumps, publishes, updates, verified = [], [], [], [], True
    finals, phase_log = [], []
    for step in range(args.warmup + args.steps):
        # ---- phase A: readers 1..N-2 pull v; the joiner comes in at 50% ----
        dc.unpublish(reader if (reader is not None and reader.is_published) else None)
        if reader is not None:
            reader.invalidate()
        dist.barrier(group=dc.pg)
        dc.replicate_start(reader if 0 < rank < joiner else None, "latest")
        if rank == 1:
            while True:
                done, nb = dc.progress(h, 0)
                if nb and done * 2 >= nb:
                    break
                time.sleep(20e-6)
        dist.barrier(group=dc.pg)  # rank 1 is half way: the joiner arrives now
        j0 = time.perf_counter()
        dc.replicate_start(h if rank == joiner else None, "latest")
        res = dc.replicate_finish(reader)
        join_s = time.perf_counter() - j0
        if reader is not None:
            assert res.status == Status.ok, res
        src_of = {a.replica: a.src for a in dc.assigns() if a.version == version}
        jl = dc.gather(join_s if rank == joiner else None)[joiner]
        # ---- phase B: version bump ----
        dist.barrier(group=dc.pg)
        b0 = time.perf_counter()
        if is_trainer:
            assert dc.unpublish(h).status == Status.ok
            m0 = time.perf_counter()
            for i, (n, v) in enumerate(views):  # new weights, in place
                ros.synth_bf16(v, 1000 * (version + 1) + i)
            torch.cuda.synchronize()
            p0 = time.perf_counter()
            assert dc.publish(h, version + 1).status == Status.ok
            pub_s = time.perf_counter() - p0
        else:
            dc.unpublish(None)
            m0 = p0 = time.perf_counter()
            dc.publish(None, version + 1)
            pub_s = 0.0
        phases = [m0 - b0, p0 - m0, time.perf_counter() - p0]
        u0 = time.perf_counter()
        pub_end = u0
        res = dc.update(reader, "latest")
        if reader is not None:
            torch.cuda.synchronize()
        # the bump ends when the last READER holds v+1 (the trainer's device
        # may still be digesting an early publish's big entries)
        t_end = time.perf_counter() if reader is not None else pub_end
        if reader is not None and not (res.status == Status.ok and res.version == version + 1):
            raise RuntimeError(f"step {step} update on {name}: {res}\n" + dc.local.trace()[-3000:])
        version += 1
        # early publish: the trainer's big-entry digests finish in the
        # background; every replica commits the final manifests before the
        # next step mutates the weights (in training, during the next step)
        fin_s = 0.0
        if early:
            dc.finalize(h if is_trainer else None)
            fin_s = time.perf_counter() - u0
        lat = dc.gather((t_end - b0, t_end - u0, pub_s, fin_s, phases))
        new_src = {a.replica: a.src for a in dc.assigns() if a.version == version}
        # v copies never serve v+1: every v+1 source is the trainer or a v+1 copy
        verified &= all(s == "trainer" or new_src.get(s) is not None for s in new_src.values())
        if not args.no_verify:
            tabs = dc.gather(table())
            verified &= len(set(tabs)) == 1
        if step >= args.warmup:
            joins.append(jl)
            bumps.append(max(x[0] for x in lat))
            updates.append(max(x[1] for x in lat))
            publishes.append(max(x[2] for x in lat))
            finals.append(max(x[3] for x in lat))
            phase_log.append([[round(y, 4) for y in x[4]] for x in lat])
    verified = all(dc.gather(verified))
    if rank == 0:
        upd = statistics.mean(updates)
        line = {
            "metric": B.METRIC, "value": round((world - 1) * total / upd / 1e9, 2), "unit": B.UNIT,
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(1e3 * statistics.mean(bumps), 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
            "config": {"workload": f"{args.workload}: elastic join + version bump (config 4): "
                                   f"trainer GPU0, readers GPU1..{world - 2} chained, joiner "
                                   f"GPU{world - 1} arrives at 50% of rollout1's batches",
                       "bytes_per_receiver": total, "receivers": world - 1, "chunk_bytes": args.chunk,
                       "join_plan": src_of, "bump_plan": new_src,
                       "l2": "inputs >> 126 MB L2; no flush"},
            "per_receiver_gbs": [round(total / upd / 1e9, 2)],
            "join_latency_s": round(statistics.mean(joins), 5),
            "bump_latency_s": round(statistics.mean(bumps), 5),
            "bump_publish_s": round(statistics.mean(publishes), 5),
            "early_publish": early,
            "bump_phases_s": {"per_rank_unpublish_mutate_publish": phase_log[-1] if phase_log else None},
            "finalize_after_update_s": round(statistics.mean(finals), 5) if early else None,
            "finalize_what": "early publish: from the readers' update call to the final manifests "
                             "committed on every registry replica (max over ranks)",
            "bump_update_s": round(upd, 5),
            "weight_update_latency_s": round(upd, 5),
            "roofline": None,
            "e2e": {"value": round((world - 1) * total / statistics.mean(bumps) / 1e9, 2),
                    "unit": B.UNIT, "h2d_bytes_per_step": None, "d2h_bytes_per_step": None,
                    "what": "unpublish + re-publish + every reader on v+1, wall clock" +
                            (" (early publish: the big-entry digests finish after the readers, "
                             "finalize_after_update_s later)" if early else " (K6 digests inside)")},
            "gpu_launches": None,
            "verified": verified,
        }
        print(json.dumps(line), flush=True)
    dist.barrier(group=dc.pg)
    dc.close()
    dist.destroy_process_group()


def run_tp2_fanout(args):
    """The north-star scenario: a TP=1 trainer (GPU0) fans Llama-3-8B out to
    TP=2 rollout replicas, resharding on pull.  Replica j's shards live on
    GPUs 2j+1 and 2j+2 (an odd last GPU holds both shards of its replica).
    All replicas replicate at once: the first reshards from the trainer, the
    next chase the first (same slicing) shard-for-shard, and so on.  Every
    receiver lands a TP-2 shard (8.03 GB).  The trainer must emit the whole
    model once, so the bound is the busiest GPU's NVLink traffic."""
    import torch
    import torch.distributed as dist

    import bench as B
    from paper_2604_09107_b200.dist import DistCluster
    from paper_2604_09107_b200.ros import Status, tp_slice

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("gloo")
    dc = DistCluster()
    shapes = B.workload_shapes(args.workload)
    total = sum(2 * B._numel(s) for _, s in shapes)
    readers = list(range(1, world))
    groups = [readers[i:i + 2] for i in range(0, len(readers), 2)]
    mine = [(j, g) for j, g in enumerate(groups) if rank in g]
    handle, shard_bufs = None, {}
    if rank == 0:
        arena, views = B.alloc_replica(shapes, dev, seed_base=42)
        handle = dc.create("m", "trainer", 1, chunk_bytes=args.chunk, pull_timeout_s=60.0)
        for (n, v), (_, shape) in zip(views, shapes):
            assert handle.register_slice(0, n, v, tp_slice(shape, 2, None, 1, 0)) == Status.ok
    elif mine:
        j, g = mine[0]
        my_shards = [0, 1] if len(g) == 1 else [g.index(rank)]
        handle = dc.create("m", f"tp2_{j}", 2, chunk_bytes=args.chunk, pull_timeout_s=60.0)
        for s in my_shards:
            for n, shape in shapes:
                geo = tp_slice(shape, 2, B.tp_dim(n), 2, s)
                buf = torch.zeros(geo[3] * geo[5], dtype=torch.uint8, device=dev)
                shard_bufs[(s, n)] = (buf, geo)
                assert handle.register_slice(s, n, buf, geo) == Status.ok
    torch.cuda.synchronize()
    dc.open(handle, endpoints=None if handle is None else
            [f"rank{rank}:cuda{local}"] * len(handle.local_shards()))
    streams = []
    if handle is not None and rank != 0:
        for s in handle.local_shards():  # a GPU holding two shards fills them concurrently
            streams.append(torch.cuda.Stream(device=dev))
            handle.set_stream(s, streams[-1])
    t0 = time.perf_counter()
    dc.publish(handle if rank == 0 else None, 1)
    publish_s = time.perf_counter() - t0
    reader = handle if rank != 0 else None

    def step():
        dc.unpublish(reader if (reader is not None and reader.is_published) else None)
        if reader is not None:
            reader.invalidate()
        dist.barrier(group=dc.pg)
        torch.cuda.synchronize()
        w0 = time.perf_counter()
        res = dc.replicate(reader, "latest")
        torch.cuda.synchronize()
        wall = time.perf_counter() - w0
        if reader is not None:
            assert res.status == Status.ok, res
            return wall, reader.stats().fill_max_ms
        return wall, 0.0

    for _ in range(args.warmup):
        step()
    verified = True
    if not args.no_verify and shard_bufs:
        for i, (n, shape) in enumerate(shapes):
            full = _synth_full(shape, 42 + i, dev)
            for s in (0, 1):
                if (s, n) in shard_bufs:
                    buf, geo = shard_bufs[(s, n)]
                    verified &= bool(torch.equal(buf, _piece(full, geo)))
            del full
    verified = all(dc.gather(verified))
    clk = B.ClockSampler(local)
    dist.barrier(group=dc.pg)
    torch.cuda.synchronize()
    clk.start()
    walls, kms = [], []
    for _ in range(args.steps):
        w, k = step()
        walls.append(w)
        kms.append(k)
    clocks = clk.stop()
    shard_bytes = {s: sum(g[3] * g[5] for (ss, n), (b, g) in shard_bufs.items() if ss == s)
                   for s in (0, 1)}
    my_bytes = sum(shard_bytes.values())
    allv = dc.gather((kms, my_bytes, sum(walls), clocks, rank))
    step_dev_ms = [max(a[0][i] for a in allv) for i in range(args.steps)]
    rx = [a for a in allv if a[1] > 0]
    total_landed = args.steps * sum(a[1] for a in rx)
    if rank == 0:
        per_rx = [round(a[1] / (statistics.mean(a[0]) / 1e3) / 1e9, 2) for a in rx]
        mean_rx = statistics.mean(per_rx)
        # busiest GPU: the trainer emits the whole model once (both halves);
        # a receiver's bound is its bytes over that time
        t_min = total / 900e9
        peaks = [a[1] / t_min / 1e9 for a in rx]
        frac = statistics.mean(x / p for x, p in zip(per_rx, peaks))
        # the same bound with the read-response protocol on the trainer's egress
        t_proto = total * (1 + B.NVL_RESP) / 900e9
        proto_frac = statistics.mean(x / (a[1] / t_proto / 1e9) for x, a in zip(per_rx, rx))
        plan = sorted({f"{a.replica}<-{a.src}" for a in dc.assigns()})
        line = {
            "metric": B.METRIC, "value": round(total_landed / (sum(step_dev_ms) / 1e3) / 1e9, 2),
            "unit": B.UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(sum(step_dev_ms) / args.steps, 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
            "config": {"workload": f"{args.workload}: TP=1 trainer (GPU0) -> {len(groups)} TP=2 "
                                   "replicas on GPU pairs, resharded on pull, chained",
                       "receivers": len(rx), "bytes_per_receiver": [a[1] for a in rx],
                       "chunk_bytes": args.chunk, "plan": plan,
                       "l2": "inputs >> 126 MB L2; no flush"},
            "per_receiver_gbs": per_rx,
            "weight_update_latency_s": round(max(a[2] for a in allv) / args.steps, 5),
            "publish_s": round(publish_s, 4),
            "roofline": {"bound": "nvlink", "achieved": round(mean_rx, 1),
                         "peak": round(statistics.mean(peaks), 1),
                         "unit": "GB/s", "frac": round(frac, 4),
                         "traffic": B.ncu_traffic("nvlink", max(a[1] for a in rx)),
                         "protocol_frac": round(proto_frac, 4),
                         "traffic_src": "NVLink bytes received per launch by the largest receiver "
                                        "(user + read-response protocol), ncu nvlrx ratio",
                         "peak_src": "per receiver: its bytes / (model bytes / 900 GB/s nominal): "
                                     "the trainer's NVLink egress carries the whole model once; "
                                     "frac = mean of achieved/peak over receivers",
                         "kernel": "pull_tma_kernel",
                         "kernel_ms_avg": round(statistics.mean(step_dev_ms), 3),
                         "alg_bytes_per_launch": max(a[1] for a in rx)},
            "e2e": {"value": round(total_landed / max(a[2] for a in allv) / 1e9, 2), "unit": B.UNIT,
                    "h2d_bytes_per_step": None, "d2h_bytes_per_step": None,
                    "what": "wall clock of the collective replicate (plan+bind+IPC exchange+kernel)"},
            "gpu_launches": args.steps * len(rx),
            "clocks": clocks,
            "verified": verified,
        }
        print(json.dumps(line), flush=True)
    dist.barrier(group=dc.pg)
    dc.close()
    dist.destroy_process_group()
