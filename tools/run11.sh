cd "$GRAFT_REPO_ROOT"
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py tests/test_gpu_serving.py -q -m gpu -s > gpurun_out/pytest_11.log 2>&1
tail -3 gpurun_out/pytest_11.log
SD_GEMM_CG=0 python tools/kbench.py --only gemm > gpurun_out/kb11_gemm.log 2>&1
python tools/kbench.py --only norm > gpurun_out/kb11_norm.log 2>&1
timeout 1200 python bench.py --steps 3 --warmup 3 > gpurun_out/bench11.json 2> gpurun_out/bench11.err
tail -3 gpurun_out/bench11.err
