# parity + config 5/2 A/B + config 3 alone
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/check_pytest.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/check_pytest.log
AB_FLAGS="--config2 1" bash tools/ab.sh main
timeout 600 python bench.py --workload config3 --steps 5 --warmup 3 --cpu-baseline 0 > gpurun_out/c3.json 2>&1; tail -1 gpurun_out/c3.json | cut -c1-300
