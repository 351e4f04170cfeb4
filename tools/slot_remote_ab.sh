# Box (tensor-map) vs slot (per-lane bulk copy) path for NVLink pulls:
# chain N=2 (one way), ring N=2 (both ways, cast) and config 3 N=2.
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
S='import json,sys; d=json.loads(sys.stdin.read()); r=d.get("roofline",{}); print(d.get("ms_per_step"), d.get("per_receiver_gbs"))'
for e in "X=1" "RSB_NO_MAPS=1"; do
  echo "== $e"
  env $e timeout 600 $T --nproc-per-node 2 --master-port 29901 bench.py --gpus 2 --no-cpu --no-host-e2e > gpurun_out/sr_c2.log 2>&1; echo c2_n2; grep '^{' gpurun_out/sr_c2.log | python -c "$S"
  env $e timeout 600 $T --nproc-per-node 2 --master-port 29902 bench.py --gpus 2 --fanout ring --workload llama3_70b_tp8 --cast --steps 10 --warmup 3 --no-cpu > gpurun_out/sr_c5.log 2>&1; echo c5_n2; grep '^{' gpurun_out/sr_c5.log | python -c "$S"
done
