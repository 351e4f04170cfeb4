# Plain peer pulls on V16 (release every batch) vs V13 for everything: chain N=4, ring N=4, c3 N=4.
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
S='import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print(d["ms_per_step"], d["per_receiver_gbs"])'
for rep in 1 2; do
for e in X=1 RSB_TMA_VARIANT=13; do
  echo "== $e"
  env $e timeout 600 $T --nproc-per-node 4 --master-port $((29990+rep)) bench.py --gpus 4 --no-cpu --no-host-e2e 2>&1 | grep "^{" | python -c "$S"
done
done
timeout 600 $T --nproc-per-node 4 --master-port 29995 bench.py --gpus 4 --fanout ring --workload llama3_70b_tp8 --cast --steps 5 --warmup 3 --no-cpu 2>&1 | grep "^{" | python -c "$S"
timeout 900 $T --nproc-per-node 4 --master-port 29996 bench.py --gpus 4 --workload qwen25_32b --reshard fsdp_tp2 --steps 5 --warmup 3 --no-cpu --no-verify 2>&1 | grep "^{" | python -c "$S"
