# 4-GPU check after V15 for cast pulls: the GPU suite and the config 5 ring at N=2/N=4
O=gpurun_out/m4v
mkdir -p $O
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 1500 python -m pytest tests -m gpu -q -rs > $O/pytest_gpu_4gpu.log 2>&1
timeout 600 $T --nproc-per-node 4 --master-port 29661 bench.py --gpus 4 --fanout ring --workload llama3_70b_tp8 --cast --steps 10 --warmup 3 --no-cpu > $O/c5_n4.log 2>&1
timeout 600 $T --nproc-per-node 2 --master-port 29662 bench.py --gpus 2 --fanout ring --workload llama3_70b_tp8 --cast --steps 10 --warmup 3 --no-cpu > $O/c5_n2.log 2>&1
