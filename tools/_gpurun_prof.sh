# round-2 profile evidence (launch list of the bench's timed region, per-class ncu metrics, conv traffic,
# one full capture of the dominant conv and dense GEMM launches)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/launches_r02.csv python bench.py --steps 1 --warmup 1 --denoise-steps 5 --profile-range \
  --no-serving --no-cpu-baseline --no-e2e --no-alt-precision > gpurun_out/launches_r02.log 2>&1; echo "launch list rc=$?"
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,launch__grid_size"
timeout 1200 ncu --metrics $M --cache-control none --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/ev_step.csv python tools/ncu_step.py > /dev/null 2>&1; echo "ev step rc=$?"
timeout 1200 ncu --metrics $M --cache-control none --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/ev_vae.csv python tools/ncu_step.py --decode > /dev/null 2>&1; echo "ev vae rc=$?"
timeout 1800 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed \
  --cache-control all --clock-control none --profile-from-start off -k regex:"gemm_kernel|splitk_reduce" --csv --page raw \
  --log-file gpurun_out/conv_cold.csv python tools/ncu_step.py > /dev/null 2>&1; echo "conv traffic rc=$?"
timeout 1800 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:gemm_kernel \
  --launch-skip 3 --launch-count 3 -o gpurun_out/gemm_full_r02 python tools/ncu_step.py > /dev/null 2>&1; echo "full rc=$?"
SD_RES_TMA=0 SD_NO_GRAPH=1 timeout 900 compute-sanitizer --tool synccheck --error-exitcode 9 python tools/sanitize_step.py tiny 8 fp16 > gpurun_out/san_synccheck_tiny_noresTMA.log 2>&1; echo "synccheck noresTMA rc=$?"
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/gputests.log 2>&1; echo "tests rc=$?"
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
