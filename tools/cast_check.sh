# fp8 cast landing: tests + config 5 N=1 (default kernel vs RSB_NO_CASTMAP-free A/B by variant)
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
J='import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print(d["ms_per_step"], r["kernel_ms_avg"], r["frac"])'
timeout 600 python bench.py --workload llama3_70b_tp8 --cast --steps 20 --warmup 3 --no-cpu > gpurun_out/castmap_c5.log 2>&1; echo "c5 cast"; grep '^{' gpurun_out/castmap_c5.log | python -c "$J" || tail -5 gpurun_out/castmap_c5.log
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu --no-host-e2e > gpurun_out/castmap_c2.log 2>&1; echo "c2"; grep '^{' gpurun_out/castmap_c2.log | python -c "$J"
