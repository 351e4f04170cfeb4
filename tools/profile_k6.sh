# Launch list of the default bench command and a --set full capture of K6
# (span_digest_kernel) on a 256 MiB item.  Each command first runs without ncu.
set -e
mkdir -p gpurun_out/pk
B="python bench.py --steps 3 --warmup 3 --no-cpu"
$B > gpurun_out/pk/bench.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/pk/launches_c2.csv $B > gpurun_out/pk/launches.log 2>&1
python tools/k6_bench.py --mb 256 > gpurun_out/pk/k6.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:span_digest -s 1 -c 1 \
    -o gpurun_out/pk/full_k6 python tools/k6_bench.py --mb 256 > gpurun_out/pk/full_k6.log 2>&1
echo profiles-done
