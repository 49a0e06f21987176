mkdir -p gpurun_out
python tools/one_egkb.py 1024 > gpurun_out/one.log 2>&1 && timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_egkb_ -s 1 -c 1 -o gpurun_out/prof_pk python tools/one_egkb.py 1024 > gpurun_out/ncu_pk.log 2>&1
tail -2 gpurun_out/ncu_pk.log
