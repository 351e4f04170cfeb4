# 4-GPU check after direct reader groups: the GPU suite and the reshard legs
O=gpurun_out/m4d2
mkdir -p $O
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 1500 python -m pytest tests -m gpu -q -rs > $O/pytest_gpu_4gpu.log 2>&1
timeout 600 $T --nproc-per-node 4 --master-port 29611 bench.py --gpus 4 --reshard tp2 --steps 8 --warmup 3 --no-cpu > $O/tp2_n4.log 2>&1
timeout 900 $T --nproc-per-node 4 --master-port 29612 bench.py --gpus 4 --workload qwen25_32b --reshard fsdp_tp2 --steps 5 --warmup 3 --no-cpu > $O/c3_n4.log 2>&1
