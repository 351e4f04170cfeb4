export RSB_DEBUG=1
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 300 python -m pytest tests/test_dist_gpu.py -x -q > gpurun_out/dist_gpu.log 2>&1; tail -1 gpurun_out/dist_gpu.log
timeout 600 $T --nproc-per-node 4 --master-port 29521 bench.py --gpus 4 --steps 10 --warmup 3 --no-cpu > gpurun_out/c2_n4.log 2>&1; tail -1 gpurun_out/c2_n4.log | cut -c1-900
timeout 600 $T --nproc-per-node 2 --master-port 29522 bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu > gpurun_out/c2_n2.log 2>&1; tail -1 gpurun_out/c2_n2.log | cut -c1-600
timeout 900 $T --nproc-per-node 4 --master-port 29523 bench.py --gpus 4 --workload qwen25_32b --reshard fsdp_tp2 --steps 5 --warmup 3 --no-cpu > gpurun_out/c3_n4.log 2>&1; tail -1 gpurun_out/c3_n4.log | cut -c1-1900
timeout 600 $T --nproc-per-node 4 --master-port 29524 bench.py --gpus 4 --fanout ring --workload llama3_70b_tp8 --cast --steps 10 --warmup 3 --no-cpu > gpurun_out/c5_n4.log 2>&1; tail -1 gpurun_out/c5_n4.log | cut -c1-900
