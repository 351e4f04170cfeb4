# NVLink pull variants on one GPU pair (diagnostic)
for cfg in "RSB_TMA_VARIANT=0" "RSB_TMA_VARIANT=2" "RSB_TMA_VARIANT=1" "RSB_NO_MAPS=1" "RSB_PULL_KERNEL=ldg"; do
  env $cfg timeout 200 python tools/p2p_probe.py "$@" 2>&1 | tail -1
done
