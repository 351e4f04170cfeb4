# Digest-chunk size sweep of the N=4 chain (config 1 and config 2): smaller
# chunks mean smaller watermark batches, so each hop's first wave lands
# sooner (diagnostic; logs in gpurun_out/cs/).
O=gpurun_out/cs
mkdir -p $O
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
p=29950
for c in 4096 2048 1024; do
  p=$((p+1)); timeout 600 $T --nproc-per-node 4 --master-port $p bench.py --gpus 4 --workload config1 --chunk $c --steps 20 --warmup 3 --no-cpu > $O/c1_c$c.log 2>&1
  p=$((p+1)); timeout 600 $T --nproc-per-node 4 --master-port $p bench.py --gpus 4 --chunk $c --steps 8 --warmup 3 --no-cpu > $O/c2_c$c.log 2>&1
done
python bench.py --chunk 2048 --steps 10 --no-cpu --no-host-e2e > $O/n1_c2048.log 2>&1
