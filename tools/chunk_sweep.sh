# Digest chunk size vs the pull kernel's roofline fraction (config 2 and 3, N=1).
for c in 2560 4096 8192 16384; do
  timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu --no-host-e2e --chunk $c > gpurun_out/chunk_c2_$c.log 2>&1
  echo "c2 chunk=$c"; grep '^{' gpurun_out/chunk_c2_$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(d['ms_per_step'], r['kernel_ms_avg'], r['frac'])"
done
for c in 8192 16384; do
  timeout 600 python bench.py --workload qwen25_32b --reshard fsdp_tp2 --steps 5 --warmup 2 --no-cpu --no-verify --chunk $c > gpurun_out/chunk_c3_$c.log 2>&1
  echo "c3 chunk=$c"; grep '^{' gpurun_out/chunk_c3_$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(d['ms_per_step'], r['kernel_ms_avg'], r['frac'])"
done
