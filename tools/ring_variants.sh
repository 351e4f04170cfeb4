# config-5-shaped ring on N GPUs (both directions of every link busy), plain vs cast, per kernel variant
N=${1:-2}
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node $N"
for v in ${2:-auto 4 5}; do
  for c in "" "--cast"; do
    if [ "$v" = auto ]; then unset RSB_TMA_VARIANT; else export RSB_TMA_VARIANT=$v; fi
    timeout 600 $T --master-port $((29600 + RANDOM % 300)) bench.py --gpus $N --fanout ring --workload llama3_70b_tp8 $c --steps 6 --warmup 3 --no-cpu --no-verify 2>/dev/null | tail -1 |
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ring N=$N v=$v ${c:-plain}', d['per_receiver_gbs'])"
  done
done
