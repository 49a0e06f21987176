# quick loop: eGKB GPU parity tests, phase trace, short bench
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/q_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/q_pytest.log
KB_PK_TRACE=1 timeout 120 python tools/one_egkb.py 1024 > gpurun_out/q_trace.log 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/q_bench.json 2> gpurun_out/q_bench.err
tail -2 gpurun_out/q_pytest.log
