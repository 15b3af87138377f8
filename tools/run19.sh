cd "$GRAFT_REPO_ROOT"
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -m gpu -x -k "attention" > gpurun_out/pytest_19.log 2>&1
tail -3 gpurun_out/pytest_19.log
for sp in 1 2; do for em in 0 3 4; do
  echo "split $sp emu $em" >> gpurun_out/kb19_attn.log
  SD_ATTN_SPLIT=$sp SD_ATTN_EMU=$em python tools/kbench.py --only attn --pick 0 2>&1 | grep attn_tc >> gpurun_out/kb19_attn.log
done; done
for em in 0 4; do
  echo "emu $em d64/d80" >> gpurun_out/kb19_attn.log
  SD_ATTN_EMU=$em python tools/kbench.py --only attn --pick 1 2>&1 | grep attn_tc >> gpurun_out/kb19_attn.log
  SD_ATTN_EMU=$em python tools/kbench.py --only attn --pick 2 2>&1 | grep attn_tc >> gpurun_out/kb19_attn.log
done
