# Round-2 profiles (one GPU): launch list of the default bench command and
# --set full captures of the fill kernel (plain config 2, the config 3
# reshard after the partial-gather change, the config 5 cast) and of K6 in
# an early publish.  Every command first runs without ncu and must exit 0.
set -e
O=gpurun_out/r2
mkdir -p $O
B="python bench.py --steps 3 --warmup 3 --no-cpu"
C="python bench.py --steps 1 --warmup 0 --no-cpu --no-verify --no-host-e2e"
$B > $O/bench.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file $O/launches_c2.csv $B > $O/ncu_launches.log 2>&1
$C > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:pull_tma -s 1 -c 1 \
    -o $O/full_plain $C > $O/ncu_full_plain.log 2>&1
R="$C --workload qwen25_32b --reshard fsdp_tp2"
$R > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:pull_tma -s 8 -c 1 \
    -o $O/full_reshard $R > $O/ncu_full_reshard.log 2>&1
K="$C --workload llama3_70b_tp8 --cast"
$K > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:pull_tma -s 1 -c 1 \
    -o $O/full_cast $K > $O/ncu_full_cast.log 2>&1
E="$C --early-publish"
$E > $O/early.log 2>&1
for r in full_plain full_reshard full_cast; do
  python tools/ncu_summary.py full $O/$r.ncu-rep > $O/$r.json
done
python tools/ncu_summary.py launches $O/launches_c2.csv > $O/launches_c2.json
echo profiles-done
