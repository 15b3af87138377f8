cd "$GRAFT_REPO_ROOT"
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -m gpu -x > gpurun_out/pytest_k9.log 2>&1
tail -15 gpurun_out/pytest_k9.log
timeout 300 python tools/kbench.py --only attn --reps 5 > gpurun_out/kb9_attn.log 2>&1
timeout 300 python tools/kbench.py --only norm > gpurun_out/kb9_norm.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -c 1 -o gpurun_out/prof_gemm320 python tools/kbench.py --only gemm --pick 3 --reps 1 > gpurun_out/ncu9a.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gn_ -c 2 -o gpurun_out/prof_gn python tools/kbench.py --only norm --pick 0 --reps 1 > gpurun_out/ncu9b.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:attn_tc -c 1 -o gpurun_out/prof_attn python tools/kbench.py --only attn --pick 0 --reps 1 > gpurun_out/ncu9c.log 2>&1
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench9.json 2> gpurun_out/bench9.err
tail -3 gpurun_out/bench9.err
