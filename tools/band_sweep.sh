# Row-block (dim 0) vs column-band (dim 1) reshard pulls on one GPU.
for d in 0 1; do
  for shp in "8192 8192" "5120 5120" "5120 27648" "27648 5120"; do
    set -- $shp
    timeout 300 python tools/band_probe.py --dim $d --rows $1 --cols $2 --tensors 24 2>&1 | tail -1
  done
done
