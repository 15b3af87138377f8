cd "$GRAFT_REPO_ROOT"
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -m gpu -x > gpurun_out/pytest_k7.log 2>&1
tail -3 gpurun_out/pytest_k7.log
SD_GEMM_CG=1 python tools/kbench.py > gpurun_out/kbench7_cg1.log 2>&1
SD_GEMM_CG=2 python tools/kbench.py > gpurun_out/kbench7_cg2.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_serving.py -q -m gpu -s > gpurun_out/pytest_p7.log 2>&1
tail -3 gpurun_out/pytest_p7.log
