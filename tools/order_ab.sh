# A/B of the interleaved multi-source batch order (RSB_BATCH_ORDER=0: batch
# order) on config 3 at N=1 and N=2, plus the reshard GPU tests.
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 600 python -m pytest tests -m gpu -x -q -k "reshard or dist" > gpurun_out/order_tests.log 2>&1; tail -2 gpurun_out/order_tests.log
for o in 1 0; do
  RSB_BATCH_ORDER=$o timeout 600 $T --nproc-per-node 2 --master-port 2981$o bench.py --gpus 2 --workload qwen25_32b --reshard fsdp_tp2 --steps 5 --warmup 3 --no-cpu > gpurun_out/c3_n2_o$o.log 2>&1
  echo "order=$o N=2"; grep '^{' gpurun_out/c3_n2_o$o.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['per_receiver_gbs'], d['roofline']['frac'])"
  RSB_BATCH_ORDER=$o timeout 600 python bench.py --workload qwen25_32b --reshard fsdp_tp2 --steps 5 --warmup 3 --no-cpu --no-host-e2e > gpurun_out/c3_n1_o$o.log 2>&1
  echo "order=$o N=1"; grep '^{' gpurun_out/c3_n1_o$o.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['frac'])"
done
