# TCP plane: socket buffer size x connections -> version-bump test pass rate
# and loopback throughput (tools/stream_probe.py, 1 GiB and Llama-3-8B).
for buf in 0 2097152 8388608; do
  for n in 2 4; do
    pass=0
    for i in 1 2 3; do
      RSB_TCP_BUF=$buf RSB_TCP_STREAMS=$n timeout 300 python -m pytest tests/test_stream.py -x -q -k version_bumps 2>&1 | tail -1 | grep -q "1 passed" && pass=$((pass+1))
    done
    g=$(RSB_TCP_BUF=$buf RSB_TCP_STREAMS=$n timeout 300 python tools/stream_probe.py --reader-dev 1 2>&1 | tail -1 | python -c "import json,sys; print(json.loads(sys.stdin.read())['gbs_wall'])" 2>/dev/null)
    echo "buf=$buf streams=$n bump_test_pass=$pass/3 gbs=$g"
  done
done
