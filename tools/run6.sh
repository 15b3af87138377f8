cd "$GRAFT_REPO_ROOT"
python tools/kbench.py > gpurun_out/kbench1.log 2>&1
timeout 900 python -m pytest tests -q -m gpu -x -s > gpurun_out/pytest_gpu.log 2>&1
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench2.json 2> gpurun_out/bench2.err
tail -3 gpurun_out/bench2.err
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -c 1 -o gpurun_out/prof_conv64 python tools/kbench.py --reps 1 --only conv > gpurun_out/ncu_conv.log 2>&1
