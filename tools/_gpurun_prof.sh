# round-2 final profile evidence: launch list of the bench's timed region, per-class ncu metrics of one
# UNet step and one decode, cold-cache conv traffic, the VAE decode time / memory at 512² and 1024²
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/launches_r02b.csv python bench.py --steps 1 --warmup 1 --denoise-steps 5 --profile-range \
  --no-serving --no-cpu-baseline --no-e2e --no-alt-precision > gpurun_out/launches_r02b.log 2>&1; echo "launch list rc=$?"
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,launch__grid_size"
timeout 1200 ncu --metrics $M --cache-control none --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/ev_step.csv python tools/ncu_step.py > /dev/null 2>&1; echo "ev step rc=$?"
timeout 1200 ncu --metrics $M --cache-control none --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/ev_vae.csv python tools/ncu_step.py --decode > /dev/null 2>&1; echo "ev vae rc=$?"
timeout 1800 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed \
  --cache-control all --clock-control none --profile-from-start off -k regex:"gemm_kernel|splitk_reduce" --csv --page raw \
  --log-file gpurun_out/conv_cold.csv python tools/ncu_step.py > /dev/null 2>&1; echo "conv traffic rc=$?"
timeout 600 python tools/vae_decode_mem.py --out gpurun_out/vae_decode_mem.json > gpurun_out/vae_decode_mem.log 2>&1; echo "vae mem rc=$?"
