cd "$GRAFT_REPO_ROOT"
python tools/kbench.py > gpurun_out/kbench8.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_serving.py -q -m gpu -s > gpurun_out/pytest_p8.log 2>&1
tail -3 gpurun_out/pytest_p8.log
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench8.json 2> gpurun_out/bench8.err
tail -3 gpurun_out/bench8.err
