O=gpurun_out/m4d
mkdir -p $O
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 600 python -m pytest tests/test_dist_gpu.py -m gpu -q > $O/pytest_dist.log 2>&1
timeout 600 $T --nproc-per-node 4 --master-port 29701 bench.py --gpus 4 --steps 10 --warmup 3 --no-cpu > $O/c2_n4.log 2>&1
timeout 600 $T --nproc-per-node 2 --master-port 29702 bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu > $O/c2_n2.log 2>&1
timeout 900 $T --nproc-per-node 4 --master-port 29703 bench.py --gpus 4 --scenario elastic --early-publish --steps 5 --warmup 2 --no-cpu > $O/c4_n4_early.log 2>&1
timeout 900 $T --nproc-per-node 4 --master-port 29704 bench.py --gpus 4 --workload qwen25_32b --reshard fsdp_tp2 --steps 5 --warmup 3 --no-cpu > $O/c3_n4.log 2>&1
timeout 600 $T --nproc-per-node 4 --master-port 29705 bench.py --gpus 4 --fanout ring --workload llama3_70b_tp8 --cast --steps 10 --warmup 3 --no-cpu > $O/c5_n4.log 2>&1
timeout 600 $T --nproc-per-node 4 --master-port 29706 bench.py --gpus 4 --workload config1 --steps 20 --warmup 3 --no-cpu > $O/c1_n4.log 2>&1
