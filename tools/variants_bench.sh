# Pull-kernel variants (RSB_TMA_VARIANT) on the bench workloads (N=1).
#   bash tools/variants_bench.sh "0 4 5 6"
for v in ${1:-0 1 2 3 4 5 6}; do
  for w in "" "--workload llama3_70b_tp8 --cast"; do
    RSB_TMA_VARIANT=$v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu $w 2>/dev/null |
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('v$v', '${w:-plain}', d['roofline']['kernel_ms_avg'], d['roofline']['frac'], d['value'])"
  done
done
