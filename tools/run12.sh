cd "$GRAFT_REPO_ROOT"
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/pytest_12.log 2>&1
tail -3 gpurun_out/pytest_12.log
python tools/kbench.py --only gemm > gpurun_out/kb12_gemm.log 2>&1
python tools/kbench.py --only conv > gpurun_out/kb12_conv.log 2>&1
python tools/kbench.py --only attn --reps 5 > gpurun_out/kb12_attn.log 2>&1
timeout 1200 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench12.json 2> gpurun_out/bench12.err
tail -3 gpurun_out/bench12.err
