cd "$GRAFT_REPO_ROOT"
mkdir -p /tmp/ncu
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -m gpu -x -k "attention" > gpurun_out/pytest_17.log 2>&1
tail -3 gpurun_out/pytest_17.log
python tools/kbench.py --only attn > gpurun_out/kb17_attn.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_tc -c 1 -o /tmp/ncu/attn \
  python tools/kbench.py --only attn --pick 0 --reps 1 > gpurun_out/ncu_attn.log 2>&1
ncu -i /tmp/ncu/attn.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > gpurun_out/attn17_source.csv.gz
ncu -i /tmp/ncu/attn.ncu-rep --page details --csv > gpurun_out/attn17_details.csv 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/pytest_17b.log 2>&1
tail -2 gpurun_out/pytest_17b.log
timeout 1200 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench17.json 2> gpurun_out/bench17.err
tail -2 gpurun_out/bench17.err
