# Static stride (V8) vs dynamic batch claiming (V13): config 2 N=1, config 3 N=1 and N=2.
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
J='import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print(d["ms_per_step"], r["kernel_ms_avg"], r["frac"], d.get("per_receiver_gbs"))'
for v in ${VARIANTS:-8 13}; do
  [ -n "$SKIP_N1" ] || RSB_TMA_VARIANT=$v timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu --no-host-e2e > gpurun_out/dyn_c2_$v.log 2>&1
  echo "c2 n1 v=$v"; grep '^{' gpurun_out/dyn_c2_$v.log | python -c "$J"
  RSB_TMA_VARIANT=$v timeout 600 python bench.py --workload qwen25_32b --reshard fsdp_tp2 --steps 5 --warmup 2 --no-cpu --no-verify > gpurun_out/dyn_c3_$v.log 2>&1
  echo "c3 n1 v=$v"; grep '^{' gpurun_out/dyn_c3_$v.log | python -c "$J"
  RSB_TMA_VARIANT=$v timeout 600 $T --nproc-per-node 2 --master-port $((29830+v)) bench.py --gpus 2 --workload qwen25_32b --reshard fsdp_tp2 --steps 5 --warmup 3 --no-cpu --no-verify > gpurun_out/dyn_c3n2_$v.log 2>&1
  echo "c3 n2 v=$v"; grep '^{' gpurun_out/dyn_c3n2_$v.log | python -c "$J"
  RSB_TMA_VARIANT=$v timeout 600 $T --nproc-per-node 2 --master-port $((29860+v)) bench.py --gpus 2 --no-cpu > gpurun_out/dyn_c2n2_$v.log 2>&1
  echo "c2 n2 v=$v"; grep '^{' gpurun_out/dyn_c2n2_$v.log | python -c "$J"
done
