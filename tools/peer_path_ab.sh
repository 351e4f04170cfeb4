# Peer segments: slot path (default) vs tensor-map boxes (RSB_PEER_BOXES=1),
# chain (config 2) and config 3 at N=4, alternating.
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
S='import json,sys; d=json.loads(sys.stdin.read()); r=d.get("roofline",{}); print(d.get("ms_per_step"), d.get("per_receiver_gbs"))'
for rep in 1 2; do
for e in X=1 RSB_PEER_BOXES=1; do
  echo "== $e rep $rep"
  env $e timeout 600 $T --nproc-per-node 4 --master-port $((29940+rep)) bench.py --gpus 4 --no-cpu --no-host-e2e > gpurun_out/pp_c2.log 2>&1; grep '^{' gpurun_out/pp_c2.log | python -c "$S"
  env $e timeout 900 $T --nproc-per-node 4 --master-port $((29950+rep)) bench.py --gpus 4 --workload qwen25_32b --reshard fsdp_tp2 --steps 5 --warmup 3 --no-cpu --no-verify > gpurun_out/pp_c3.log 2>&1; grep '^{' gpurun_out/pp_c3.log | python -c "$S"
done
done
