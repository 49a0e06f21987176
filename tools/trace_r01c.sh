mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/sync_probe tools/sync_probe.cu && timeout 60 /tmp/sync_probe > gpurun_out/sync_probe.log 2>&1
KB_PK_TRACE=1 timeout 120 python tools/one_egkb.py 1024 > gpurun_out/pk_trace.log 2>&1
KB_PK_TRACE=1 timeout 120 python tools/ra_trace.py > gpurun_out/ra_trace.log 2>&1
nvidia-smi -q | grep -i -A3 "L2\|Max Clocks" | head -20 > gpurun_out/smi.log
