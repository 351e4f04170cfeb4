import sys, time, os
sys.path.insert(0, os.getcwd())
import torch
import bench as B
from paper_2604_09107_b200.ros import Cluster, Status
dev = torch.device("cuda:0")
shapes = B.workload_shapes("qwen25_32b")
tarena, tviews = B.alloc_replica(shapes, dev, seed_base=42)
rarena, rviews = B.alloc_replica(shapes, dev)
cl = Cluster()
t = cl.open("m", "trainer", 8); r = cl.open("m", "rollout1", 2)
B.register_pair(t, r, shapes, tviews, rviews, dev, True, False)
s = torch.cuda.Stream()
for k in range(2): r.set_stream(k, s)
assert t.publish(1).status == Status.ok
for i in range(6):
    ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ea.record(s)
    t0 = time.perf_counter()
    if r.is_published: r.unpublish()
    t1 = time.perf_counter()
    r.invalidate()
    t2 = time.perf_counter()
    res = r.replicate("latest")
    t3 = time.perf_counter()
    eb.record(s); eb.synchronize()
    st = r.stats()
    print(f"unpub {1e3*(t1-t0):.3f} inval {1e3*(t2-t1):.3f} repl {1e3*(t3-t2):.3f} dev {ea.elapsed_time(eb):.3f} fills {st.fill_sum_ms:.3f}", flush=True)
