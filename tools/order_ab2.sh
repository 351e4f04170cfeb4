# Link-class interleave (default) vs batch order (RSB_BATCH_ORDER=0), with the
# dynamic-claim kernel: config 3 at N=2 and N=1.
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
J='import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print(d["ms_per_step"], r["kernel_ms_avg"], r["frac"], d.get("per_receiver_gbs"))'
for o in 1 0; do
  RSB_BATCH_ORDER=$o timeout 600 $T --nproc-per-node 2 --master-port $((29850+o)) bench.py --gpus 2 --workload qwen25_32b --reshard fsdp_tp2 --steps 5 --warmup 3 --no-cpu > gpurun_out/o2_c3n2_$o.log 2>&1
  echo "c3 n2 order=$o"; grep '^{' gpurun_out/o2_c3n2_$o.log | python -c "$J"
done
RSB_BATCH_ORDER=1 timeout 600 python bench.py --workload qwen25_32b --reshard fsdp_tp2 --steps 5 --warmup 2 --no-cpu --no-verify > gpurun_out/o2_c3n1.log 2>&1
echo "c3 n1"; grep '^{' gpurun_out/o2_c3n1.log | python -c "$J"
