KB_PK_TRACE=1 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-sweep > gpurun_out/b.json 2> gpurun_out/b.err
grep "pk phases" gpurun_out/b.err | head -14 | awk '{s=0; for(i=4;i<=NF;i++) s+=$i; printf "%.0f ", s}'
echo
tail -c 300 gpurun_out/b.json
