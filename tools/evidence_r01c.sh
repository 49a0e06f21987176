# Round-1 evidence refresh (tiled eGKB, tiled R(A) block product, host SVD of C)
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/ev_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ev_pytest.log
timeout 300 python __graft_entry__.py > gpurun_out/ev_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/ev_smoke.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r01.json 2> gpurun_out/bench_r01.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_r01.json 2> gpurun_out/bench_ref_r01.err
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_r01.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/ncu_launch.log 2>&1
python tools/one_egkb.py 1024 > gpurun_out/one.log 2>&1 && timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_egkb_tiled -s 1 -c 1 -o gpurun_out/prof_egkb_tiled_r01 python tools/one_egkb.py 1024 > gpurun_out/ncu_egkb.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_rat_ -s 8 -c 4 -o gpurun_out/prof_rat_r01 python tools/ra_trace.py > gpurun_out/ncu_rat.log 2>&1
python tools/kron_apply_one.py > gpurun_out/kron_one.log 2>&1 && timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_dgemm -s 4 -c 4 -o gpurun_out/prof_dgemm_r01 python tools/kron_apply_one.py > gpurun_out/ncu_dgemm.log 2>&1
ls -la gpurun_out
