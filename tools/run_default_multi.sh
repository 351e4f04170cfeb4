T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 600 $T --nproc-per-node 4 --master-port 29701 bench.py --gpus 4 > gpurun_out/c2_n4_default.log 2>&1; tail -1 gpurun_out/c2_n4_default.log | cut -c1-700
timeout 600 $T --nproc-per-node 4 --master-port 29702 bench.py --impl reference --gpus 4 --steps 3 --warmup 1 > gpurun_out/ref_n4.log 2>&1; tail -1 gpurun_out/ref_n4.log | cut -c1-600
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ref_n1.log 2>&1; tail -1 gpurun_out/ref_n1.log | cut -c1-600
