# Default kernel (V13) checks: GPU tests, smoke, config 5 cast at N=1, config 2 N=1.
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
J='import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print(d["ms_per_step"], r["kernel_ms_avg"], r["frac"], d.get("e2e",{}).get("value"))'
for v in 8 13; do
RSB_TMA_VARIANT=$v timeout 600 python bench.py --workload llama3_70b_tp8 --cast --steps 20 --warmup 3 --no-cpu > gpurun_out/v13_c5_$v.log 2>&1; echo "c5 cast v=$v"; grep '^{' gpurun_out/v13_c5_$v.log | python -c "$J"
done
timeout 600 python bench.py > gpurun_out/v13_default.log 2>&1; echo default; grep '^{' gpurun_out/v13_default.log | python -c "$J"
