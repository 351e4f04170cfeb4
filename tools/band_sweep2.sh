# Row-block vs column-band reshard pulls across NVLink (trainer on cuda:1).
for d in 0 1; do
  for shp in "5120 27648" "27648 5120" "8192 8192"; do
    set -- $shp
    timeout 300 python tools/band_probe.py --src-dev 1 --dim $d --rows $1 --cols $2 --tensors 24 2>&1 | tail -1
  done
done
