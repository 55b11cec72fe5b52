# GPU parity suite + A/B of the given library variants (tools/ab.sh)
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/check_pytest.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/check_pytest.log
bash tools/ab.sh "$@"
