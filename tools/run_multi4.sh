# 4-GPU measurements of every multi-GPU bench leg (one call), then the GPU tests.
export RSB_DEBUG=1
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
S='import json,sys; d=json.loads(sys.stdin.read()); r=d.get("roofline",{}); print(d.get("ms_per_step"), d.get("per_receiver_gbs"), r.get("frac"), r.get("protocol_frac"))'
timeout 600 $T --nproc-per-node 4 --master-port 29801 bench.py --gpus 4 --no-cpu > gpurun_out/c2_n4.log 2>&1; echo c2_n4; grep '^{' gpurun_out/c2_n4.log | python -c "$S"
timeout 900 $T --nproc-per-node 4 --master-port 29802 bench.py --gpus 4 --workload qwen25_32b --reshard fsdp_tp2 --steps 5 --warmup 3 --no-cpu > gpurun_out/c3_n4.log 2>&1; echo c3_n4; grep '^{' gpurun_out/c3_n4.log | python -c "$S"
timeout 900 $T --nproc-per-node 4 --master-port 29803 bench.py --gpus 4 --scenario elastic --steps 3 --warmup 1 --no-cpu > gpurun_out/c4_n4.log 2>&1; echo c4_n4; grep '^{' gpurun_out/c4_n4.log | cut -c1-600
timeout 600 $T --nproc-per-node 4 --master-port 29804 bench.py --gpus 4 --fanout ring --workload llama3_70b_tp8 --cast --steps 10 --warmup 3 --no-cpu > gpurun_out/c5_n4.log 2>&1; echo c5_n4; grep '^{' gpurun_out/c5_n4.log | python -c "$S"
timeout 600 $T --nproc-per-node 4 --master-port 29805 bench.py --gpus 4 --reshard tp2 --steps 8 --warmup 3 --no-cpu > gpurun_out/tp2_n4.log 2>&1; echo tp2_n4; grep '^{' gpurun_out/tp2_n4.log | python -c "$S"
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
