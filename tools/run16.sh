cd "$GRAFT_REPO_ROOT"
mkdir -p /tmp/ncu
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py -q -m gpu -x -s > gpurun_out/pytest_16.log 2>&1
tail -3 gpurun_out/pytest_16.log
python tools/kbench.py --only conv > gpurun_out/kb16_conv.log 2>&1
SD_CONV_CG_OLD=1 python tools/kbench.py --only conv > gpurun_out/kb16_conv_old.log 2>&1
python tools/kbench.py --only vae > gpurun_out/kb16_vae.log 2>&1
SD_CONV_CG_OLD=1 python tools/kbench.py --only vae > gpurun_out/kb16_vae_old.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_tc -c 1 -o /tmp/ncu/attn \
  python tools/kbench.py --only attn --pick 0 --reps 1 > gpurun_out/ncu_attn.log 2>&1
ncu -i /tmp/ncu/attn.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > gpurun_out/attn_source.csv.gz
ncu -i /tmp/ncu/attn.ncu-rep --page details --csv > gpurun_out/attn_details.csv 2>&1
ncu -i /tmp/ncu/attn.ncu-rep --page raw --csv | gzip > gpurun_out/attn_raw.csv.gz
ls -la gpurun_out
