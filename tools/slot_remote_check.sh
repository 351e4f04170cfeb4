# Peer segments on the slot path: config 3 N=2, chain N=2, ring N=2, host e2e N=1, tests.
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
S='import json,sys; d=json.loads(sys.stdin.read()); r=d.get("roofline",{}); print(d.get("ms_per_step"), d.get("per_receiver_gbs"), r.get("frac"), (d.get("e2e") or {}).get("value"))'
timeout 300 python tools/mix_probe.py --mode both 2>&1 | tail -1
timeout 600 $T --nproc-per-node 2 --master-port 29911 bench.py --gpus 2 --workload qwen25_32b --reshard fsdp_tp2 --steps 5 --warmup 3 --no-cpu > gpurun_out/src_c3.log 2>&1; echo c3_n2; grep '^{' gpurun_out/src_c3.log | python -c "$S"
timeout 600 $T --nproc-per-node 2 --master-port 29912 bench.py --gpus 2 --no-cpu > gpurun_out/src_c2.log 2>&1; echo c2_n2; grep '^{' gpurun_out/src_c2.log | python -c "$S"
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/src_c2n1.log 2>&1; echo c2_n1; grep '^{' gpurun_out/src_c2n1.log | python -c "$S"
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
