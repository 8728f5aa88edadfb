nvidia-smi -q -d POWER | grep -i "limit\|draw" | head -12
python tools/micro/ab.py 3d27pt tc "stencil_tc3d_hybrid=0" > /dev/null 2>&1 &
P=$!
AB_ROUNDS=40 python tools/micro/ab.py 3d27pt tc "stencil_tc3d_hybrid=0" > /dev/null 2>&1 &
sleep 6
for i in 1 2 3 4 5 6 7 8; do nvidia-smi --query-gpu=clocks.sm,clocks.mem,power.draw,temperature.gpu,clocks_throttle_reasons.active,clocks_event_reasons.sw_power_cap,clocks_event_reasons.hw_slowdown --format=csv,noheader; sleep 0.5; done
wait
