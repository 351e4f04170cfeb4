# Config 3 at N=2: pull-kernel shape variants (RSB_TMA_VARIANT) on the mixed
# local + NVLink reshard fill.
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for v in 8 4 9 10 0; do
  RSB_TMA_VARIANT=$v timeout 600 $T --nproc-per-node 2 --master-port 2982$v bench.py --gpus 2 --workload qwen25_32b --reshard fsdp_tp2 --steps 5 --warmup 3 --no-cpu --no-verify > gpurun_out/c3v_$v.log 2>&1
  echo "variant=$v"; grep '^{' gpurun_out/c3v_$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['per_receiver_gbs'], d['roofline']['frac'])"
done
