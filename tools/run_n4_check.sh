mkdir -p gpurun_out/v4
CUDA_VISIBLE_DEVICES=0 python -m pytest tests -m gpu -x -q > gpurun_out/v4/pytest_gpu_1gpu.log 2>&1; echo "rc=$?" >> gpurun_out/v4/pytest_gpu_1gpu.log
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 4 > gpurun_out/v4/bench_n4.log 2>&1; echo "rc=$?" >> gpurun_out/v4/bench_n4.log
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29513 bench.py --impl reference --gpus 4 > gpurun_out/v4/ref_n4.log 2>&1; echo "rc=$?" >> gpurun_out/v4/ref_n4.log
for f in gpurun_out/v4/*.log; do echo "== $f"; tail -n 2 $f | cut -c1-400; done
