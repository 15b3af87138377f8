cd "$GRAFT_REPO_ROOT"
mkdir -p /tmp/ncu
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -m gpu -x -k "attention" > gpurun_out/pytest_18.log 2>&1
tail -3 gpurun_out/pytest_18.log
python tools/kbench.py --only attn > gpurun_out/kb18_attn.log 2>&1
SD_ATTN_SPLIT=1 python tools/kbench.py --only attn --pick 0 > gpurun_out/kb18_attn_s1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_tc -c 1 -o /tmp/ncu/attn \
  python tools/kbench.py --only attn --pick 0 --reps 1 > gpurun_out/ncu_attn.log 2>&1
ncu -i /tmp/ncu/attn.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > gpurun_out/attn18_source.csv.gz
ncu -i /tmp/ncu/attn.ncu-rep --page details --csv > gpurun_out/attn18_details.csv 2>&1
