# Config 3 (N=1, FSDP-8 -> TP-2 reshard on one GPU): plan statistics and one
# --set full capture of a steady-state fill kernel.
set -e
C="python bench.py --workload qwen25_32b --reshard fsdp_tp2 --steps 1 --warmup 1 --no-cpu --no-verify --no-host-e2e"
$C > gpurun_out/c3_plain.log 2>&1

ncu --set full --clock-control none --import-source on -k regex:pull_tma -s 9 -c 1 \
    -o gpurun_out/full_c3 $C > gpurun_out/prof_full_c3.log 2>&1
echo done
