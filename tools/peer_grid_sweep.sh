O=gpurun_out/pg
mkdir -p $O
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
p=29900
for g in 0 96 64 40; do
  p=$((p+1)); RSB_PEER_GRID=$g timeout 600 $T --nproc-per-node 4 --master-port $p bench.py --gpus 4 --workload config1 --steps 20 --warmup 3 --no-cpu > $O/c1_g$g.log 2>&1
  p=$((p+1)); RSB_PEER_GRID=$g timeout 600 $T --nproc-per-node 4 --master-port $p bench.py --gpus 4 --steps 8 --warmup 3 --no-cpu > $O/c2_g$g.log 2>&1
done
