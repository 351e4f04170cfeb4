# Config 3 at N=1 (FSDP-8 -> TP-2 on one GPU): pull-kernel shape variants.
for v in 8 7 9 10 4 0; do
  RSB_TMA_VARIANT=$v timeout 600 python bench.py --workload qwen25_32b --reshard fsdp_tp2 --steps 5 --warmup 2 --no-cpu --no-verify > gpurun_out/c3n1v_$v.log 2>&1
  echo "variant=$v"; grep '^{' gpurun_out/c3n1v_$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(d['ms_per_step'], r['kernel_ms_avg'], r['frac'])"
done
