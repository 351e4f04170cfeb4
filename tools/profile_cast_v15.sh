# --set full capture of the fused-cast pull (V15 shape) of config 5; the
# command runs without ncu first.
set -e
O=gpurun_out/pc
mkdir -p $O
C="python bench.py --steps 1 --warmup 0 --no-cpu --no-verify --no-host-e2e"
K="$C --workload llama3_70b_tp8 --cast"
$K > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:pull_tma -s 1 -c 1 \
    -o $O/full_cast_v15 $K > $O/ncu_full_cast_v15.log 2>&1
for r in full_cast_v15; do
  python tools/ncu_summary.py full $O/$r.ncu-rep > $O/$r.json
done
echo profiles-done
