# round evidence for the current build: parity suite, default bench line, reference arm,
# config-5 launch list (one step, serialised) and config-2 launch list
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/final_pytest.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/final_pytest.log
timeout 900 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; echo bench_rc=$?
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/final_ref.json 2>&1; echo ref_rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/final_launches_c5.csv python tools/profile_step.py > /dev/null 2>&1; echo ncu5_rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/final_launches_c2.csv python tools/profile_step.py 512 0.0016914558667664816 > /dev/null 2>&1; echo ncu2_rc=$?
