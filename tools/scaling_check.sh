# The driver's scaling commands at N=1,2,4 (default config) and the reference arm at N=4.
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
S='import json,sys; d=json.loads(sys.stdin.read()); print(d.get("n_gpus"), d.get("value"), d.get("ms_per_step"), (d.get("e2e") or {}).get("value"), d.get("gpu_launches"), d.get("clocks",{}).get("reasons"))'
timeout 900 python bench.py 2>&1 | grep "^{" | python -c "$S"
timeout 900 $T --nproc-per-node 2 --master-port 29981 bench.py --gpus 2 2>&1 | grep "^{" | python -c "$S"
timeout 900 $T --nproc-per-node 4 --master-port 29982 bench.py --gpus 4 2>&1 | grep "^{" | python -c "$S"
timeout 900 $T --nproc-per-node 4 --master-port 29983 bench.py --impl reference --gpus 4 2>&1 | grep "^{" | cut -c1-300
