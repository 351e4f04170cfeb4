# 4-GPU check after the member-cut chunk change: the GPU suite and the
# reshard / chain legs (logs in gpurun_out/m4c/).
O=gpurun_out/m4c
mkdir -p $O
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 1500 python -m pytest tests -m gpu -q -rs > $O/pytest_gpu_4gpu.log 2>&1
timeout 900 $T --nproc-per-node 4 --master-port 29601 bench.py --gpus 4 --workload qwen25_32b --reshard fsdp_tp2 --steps 5 --warmup 3 --no-cpu > $O/c3_n4.log 2>&1
timeout 600 $T --nproc-per-node 2 --master-port 29602 bench.py --gpus 2 --workload qwen25_32b --reshard fsdp_tp2 --steps 5 --warmup 3 --no-cpu > $O/c3_n2.log 2>&1
timeout 600 $T --nproc-per-node 4 --master-port 29603 bench.py --gpus 4 --reshard tp2 --steps 8 --warmup 3 --no-cpu > $O/tp2_n4.log 2>&1
timeout 600 $T --nproc-per-node 4 --master-port 29604 bench.py --gpus 4 --steps 10 --warmup 3 --no-cpu > $O/c2_n4.log 2>&1
