# Final 4-GPU refresh of every multi-GPU bench leg (one call); logs in
# gpurun_out/m4f/ (copied to profiles/r2/multi_final/ afterwards).
O=gpurun_out/m4f
mkdir -p $O
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 600 $T --nproc-per-node 2 --master-port 29800 bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu > $O/c2_n2.log 2>&1
timeout 600 $T --nproc-per-node 4 --master-port 29801 bench.py --gpus 4 --steps 10 --warmup 3 --no-cpu > $O/c2_n4.log 2>&1
timeout 600 $T --nproc-per-node 4 --master-port 29808 bench.py --gpus 4 --workload config1 --steps 20 --warmup 3 --no-cpu > $O/c1_n4.log 2>&1
timeout 600 python bench.py --workload config1 --steps 20 --warmup 3 --no-cpu > $O/c1_n1.log 2>&1
timeout 900 $T --nproc-per-node 4 --master-port 29802 bench.py --gpus 4 --workload qwen25_32b --reshard fsdp_tp2 --steps 5 --warmup 3 --no-cpu > $O/c3_n4.log 2>&1
timeout 900 $T --nproc-per-node 4 --master-port 29803 bench.py --gpus 4 --scenario elastic --steps 5 --warmup 2 --no-cpu > $O/c4_n4.log 2>&1
timeout 900 $T --nproc-per-node 4 --master-port 29806 bench.py --gpus 4 --scenario elastic --early-publish --steps 5 --warmup 2 --no-cpu > $O/c4_n4_early.log 2>&1
timeout 600 $T --nproc-per-node 4 --master-port 29804 bench.py --gpus 4 --fanout ring --workload llama3_70b_tp8 --cast --steps 10 --warmup 3 --no-cpu > $O/c5_n4.log 2>&1
timeout 600 $T --nproc-per-node 4 --master-port 29805 bench.py --gpus 4 --reshard tp2 --steps 8 --warmup 3 --no-cpu > $O/tp2_n4.log 2>&1
timeout 900 $T --nproc-per-node 4 --master-port 29807 bench.py --impl reference --gpus 4 --steps 2 --warmup 1 > $O/ref_n4.log 2>&1
echo multi-done
