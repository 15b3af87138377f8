cd "$GRAFT_REPO_ROOT"
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/launches_r01.csv python bench.py --steps 1 --warmup 3 --no-serving --no-e2e \
  --no-cpu-baseline --profile-range > gpurun_out/ncu_list.log 2>&1
echo "list rc=$?"
SD_NO_GRAPH=1 SD_NVTX=1 timeout 1200 ncu --set full --clock-control none --import-source on --profile-from-start off \
  --nvtx --nvtx-include "conv/" -o gpurun_out/conv_full python tools/ncu_step.py > gpurun_out/ncu_conv.log 2>&1
echo "conv rc=$?"
SD_NO_GRAPH=1 SD_NVTX=1 timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
  --nvtx --nvtx-include "gemm/" -c 60 -o gpurun_out/gemm_full python tools/ncu_step.py > gpurun_out/ncu_gemm.log 2>&1
echo "gemm rc=$?"
timeout 1200 python bench.py > gpurun_out/bench14.json 2> gpurun_out/bench14.err
echo "bench rc=$?"
tail -2 gpurun_out/bench14.err
