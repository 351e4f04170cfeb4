# Watermark release group size: V8 (4 batches per sys fence), V11 (8), V12 (16)
# on config 2 N=1 and config 3 N=1.
for v in 8 11 12; do
  RSB_TMA_VARIANT=$v timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu --no-host-e2e > gpurun_out/relv_c2_$v.log 2>&1
  echo "c2 variant=$v"; grep '^{' gpurun_out/relv_c2_$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(d['ms_per_step'], r['kernel_ms_avg'], r['frac'])"
  RSB_TMA_VARIANT=$v timeout 600 python bench.py --workload qwen25_32b --reshard fsdp_tp2 --steps 5 --warmup 2 --no-cpu --no-verify > gpurun_out/relv_c3_$v.log 2>&1
  echo "c3 variant=$v"; grep '^{' gpurun_out/relv_c3_$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(d['ms_per_step'], r['kernel_ms_avg'], r['frac'])"
done
