python tools/one_egkb.py 1024 > gpurun_out/one.log 2>&1 && timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_egkb_persistent -s 1 -c 1 -o gpurun_out/prof_egkb_r01 python tools/one_egkb.py 1024 > gpurun_out/ncu_egkb.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_ra_block -s 2 -c 1 -o gpurun_out/prof_rablock_r01 python tools/ra_probe.py > gpurun_out/ncu_ra.log 2>&1
tail -n 2 gpurun_out/ncu_egkb.log gpurun_out/ncu_ra.log
