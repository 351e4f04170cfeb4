# Re-check after a K6 change: full GPU suite, smoke, N=1 bench, K6 micro, config 4 at N=4.
mkdir -p gpurun_out/fk
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
python -m pytest tests -m gpu -x -q > gpurun_out/fk/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/fk/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/fk/smoke.log 2>&1
python bench.py > gpurun_out/fk/bench_n1.log 2>&1
python tools/k6_bench.py --mb 1024 > gpurun_out/fk/k6.log 2>&1
python tools/k6_bench.py --mb 1024 >> gpurun_out/fk/k6.log 2>&1
RSB_TIMING=1 timeout 900 $T --nproc-per-node 4 --master-port 29803 bench.py --gpus 4 --scenario elastic --steps 3 --warmup 1 --no-cpu > gpurun_out/fk/bench_c4_n4.log 2>&1
for f in gpurun_out/fk/*.log; do echo "== $f"; tail -n 2 $f | cut -c1-300; done
