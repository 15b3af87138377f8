cd "$GRAFT_REPO_ROOT"
for nb in 1 2; do for sp in 1 2; do
  echo "nb $nb split $sp" >> gpurun_out/kb20_attn.log
  SD_ATTN_NB=$nb SD_ATTN_SPLIT=$sp SD_ATTN_EMU=0 python tools/kbench.py --only attn --pick 0 2>&1 | grep attn_tc >> gpurun_out/kb20_attn.log
done; done
SD_ATTN_NB=2 SD_ATTN_SPLIT=2 timeout 600 python -m pytest tests/test_gpu_kernels.py -q -m gpu -x -k "attention" > gpurun_out/pytest_20.log 2>&1
tail -1 gpurun_out/pytest_20.log
