# Copy-engine landing of host sources: retention tests, host e2e (N=1), offload probe, A/B.
S='import json,sys; d=json.loads(sys.stdin.read()); print(d["e2e"]["value"], d["roofline"]["frac"])'
timeout 600 python -m pytest tests/test_retention.py tests/test_gpu_client.py -x -q 2>&1 | tail -1
for e in X=1 RSB_HOST_DMA=0; do echo "== $e"; env $e timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu 2>&1 | tail -1 | python -c "$S"; env $e timeout 300 python tools/offload_probe.py 2>&1 | tail -1 | cut -c1-300; done
