# Config 3 N=1 step breakdown: host phase times (RSB_TIMING) and the bench line.
RSB_TIMING=1 timeout 600 python bench.py --workload qwen25_32b --reshard fsdp_tp2 --steps 3 --warmup 2 --no-cpu --no-verify > gpurun_out/c3_timing.log 2>&1
grep '\[rsb\]' gpurun_out/c3_timing.log | tail -16
grep '^{' gpurun_out/c3_timing.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], json.dumps(d['roofline']))"
