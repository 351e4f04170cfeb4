# ncu NVLink counters of a pull on GPU0 while GPU1 pulls from GPU0 in another
# process (both directions of GPU0's port busy).  Output: gpurun_out/bc/.
O=gpurun_out/bc
mkdir -p $O
python tools/bidir_counters.py --profiled > $O/alone.log 2>&1   # warm + one-way reference timing
python tools/bidir_counters.py --background 150 > $O/background.log 2>&1 &
BG=$!
sleep 25
M=gpu__time_duration.sum,nvlrx__bytes.sum,nvlrx__bytes_data_user.sum,nvlrx__bytes_data_protocol.sum,nvlrx__bytes_packet_request.sum,nvlrx__bytes_packet_response.sum,nvltx__bytes.sum,nvltx__bytes_data_user.sum,nvltx__bytes_data_protocol.sum,nvltx__bytes_packet_request.sum,nvltx__bytes_packet_response.sum
timeout 600 ncu --metrics $M --clock-control none --kernel-name regex:pull_tma --csv --log-file $O/counters.csv python tools/bidir_counters.py --profiled > $O/profiled.log 2>&1
timeout 600 ncu --metrics $M --clock-control none --kernel-name regex:pull_tma --csv --log-file $O/counters_alone.csv python tools/bidir_counters.py --profiled > $O/profiled_alone_during_bg_end.log 2>&1
wait $BG
timeout 600 ncu --metrics $M --clock-control none --kernel-name regex:pull_tma --csv --log-file $O/counters_oneway.csv python tools/bidir_counters.py --profiled > $O/profiled_oneway.log 2>&1
