# End-of-round refresh on 2 GPUs: GPU tests, smoke, the default bench and the
# reference arm at N=1 and N=2, then the ncu launch list + full captures.
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
mkdir -p gpurun_out/final
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/final/pytest_gpu.log 2>&1; tail -1 gpurun_out/final/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/final/smoke.log 2>&1; tail -1 gpurun_out/final/smoke.log
timeout 900 python bench.py > gpurun_out/final/bench_n1.log 2>&1; tail -1 gpurun_out/final/bench_n1.log | cut -c1-200
timeout 900 python bench.py --impl reference > gpurun_out/final/ref_n1.log 2>&1; tail -1 gpurun_out/final/ref_n1.log | cut -c1-200
timeout 900 $T --nproc-per-node 2 --master-port 29931 bench.py --gpus 2 > gpurun_out/final/bench_n2.log 2>&1; tail -1 gpurun_out/final/bench_n2.log | cut -c1-200
timeout 900 $T --nproc-per-node 2 --master-port 29932 bench.py --impl reference --gpus 2 > gpurun_out/final/ref_n2.log 2>&1; tail -1 gpurun_out/final/ref_n2.log | cut -c1-200
bash tools/profile_round.sh
