# Round profiles (one GPU): launch list of the default bench command and
# --set full captures of the fill kernel, plain and fp8-cast.  Each command
# first runs without ncu and must exit 0.
set -e
B="python bench.py --steps 3 --warmup 3 --no-cpu"
C="python bench.py --steps 1 --warmup 0 --no-cpu --no-verify"
$B > gpurun_out/prof_bench.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/launches_c2.csv $B > gpurun_out/prof_launches.log 2>&1
$C > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:pull_tma -s 1 -c 1 \
    -o gpurun_out/full_plain $C > gpurun_out/prof_full_plain.log 2>&1
$C --workload llama3_70b_tp8 --cast > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:pull_tma -s 1 -c 1 \
    -o gpurun_out/full_cast $C --workload llama3_70b_tp8 --cast > gpurun_out/prof_full_cast.log 2>&1
echo profiles-done
