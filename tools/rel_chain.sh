# Watermark release group vs chain hop efficiency (config 2 at N=4).
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
S='import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print(d["ms_per_step"], d["per_receiver_gbs"], r.get("protocol_frac"))'
for v in 13 16 17 13 16 17; do
  echo "v=$v"; RSB_TMA_VARIANT=$v timeout 600 $T --nproc-per-node 4 --master-port $((29970+v)) bench.py --gpus 4 --no-cpu --no-host-e2e 2>&1 | grep "^{" | python -c "$S"
done
