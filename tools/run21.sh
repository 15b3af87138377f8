cd "$GRAFT_REPO_ROOT"
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -s -k "xl" > gpurun_out/pytest_21xl.log 2>&1
tail -12 gpurun_out/pytest_21xl.log
timeout 1500 python -m pytest tests/ -q -m gpu -x > gpurun_out/pytest_21.log 2>&1
tail -3 gpurun_out/pytest_21.log
