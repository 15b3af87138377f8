cd "$GRAFT_REPO_ROOT"
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -m gpu > gpurun_out/pytest_k10.log 2>&1
tail -5 gpurun_out/pytest_k10.log
for m in 0 1 2 3 4; do echo "dbg=$m"; SD_EPI_DBG=$m SD_GEMM_CG=1 python tools/kbench.py --only gemm --reps 20; done > gpurun_out/kb10_epi.log 2>&1
timeout 900 python -m pytest tests/test_gpu_serving.py -q -m gpu -s > gpurun_out/pytest_s10.log 2>&1
tail -3 gpurun_out/pytest_s10.log
