cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py tests/test_gpu_serving.py -q -m gpu -x > gpurun_out/pytest_13.log 2>&1
tail -3 gpurun_out/pytest_13.log
python tools/kbench.py --only conv > gpurun_out/kb13_conv.log 2>&1
SD_SPLITK=1 python tools/kbench.py --only conv > gpurun_out/kb13_conv_nosplit.log 2>&1
SD_SPLITK=2 python tools/kbench.py --only conv > gpurun_out/kb13_conv_s2.log 2>&1
SD_SPLITK=4 python tools/kbench.py --only conv > gpurun_out/kb13_conv_s4.log 2>&1
timeout 1200 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench13.json 2> gpurun_out/bench13.err
tail -3 gpurun_out/bench13.err
