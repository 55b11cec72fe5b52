set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2s2_pytest.log 2>&1; echo pytest_rc=$? >> gpurun_out/r2s2_pytest.log
tail -3 gpurun_out/r2s2_pytest.log
timeout 900 python bench.py > gpurun_out/r2s2_bench.json 2> gpurun_out/r2s2_bench.err; echo bench_rc=$?
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2s2_ref.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2s2_launches.csv python tools/profile_step.py > gpurun_out/r2s2_ncu.log 2>&1; echo ncu_rc=$?
for t in memcheck racecheck synccheck; do timeout 600 compute-sanitizer --tool $t --error-exitcode 9 python tools/sanitize_step.py > gpurun_out/r2s2_san_$t.log 2>&1; echo san_$t=$?; done
