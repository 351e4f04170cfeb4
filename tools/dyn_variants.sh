# Dynamic-claim kernel shapes (V13 2x512 B stages, V14 4x256 B, V15 3x512 B):
# config 3 at N=2 (mixed local + NVLink) and config 2 at N=1.
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
J='import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print(d["ms_per_step"], r["kernel_ms_avg"], r["frac"], d.get("per_receiver_gbs"))'
for v in 13 14 15; do
  RSB_TMA_VARIANT=$v timeout 600 $T --nproc-per-node 2 --master-port $((29880+v)) bench.py --gpus 2 --workload qwen25_32b --reshard fsdp_tp2 --steps 5 --warmup 3 --no-cpu --no-verify > gpurun_out/dv_c3n2_$v.log 2>&1
  echo "c3 n2 v=$v"; grep '^{' gpurun_out/dv_c3n2_$v.log | python -c "$J"
  RSB_TMA_VARIANT=$v timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu --no-host-e2e > gpurun_out/dv_c2_$v.log 2>&1
  echo "c2 n1 v=$v"; grep '^{' gpurun_out/dv_c2_$v.log | python -c "$J"
done
