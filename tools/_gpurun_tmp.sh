mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 1300 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 900 python bench.py > gpurun_out/bench_final3.log 2> gpurun_out/bench_final3.err; tail -c 3000 gpurun_out/bench_final3.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 1 --warmup 3 --denoise-steps 5 --profile-range --no-cpu-baseline --no-e2e --no-serving > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,launch__grid_size --cache-control none --clock-control none --profile-from-start off --csv --log-file gpurun_out/ev_step.csv python tools/ncu_step.py > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,launch__grid_size --cache-control none --clock-control none --profile-from-start off --csv --log-file gpurun_out/ev_vae.csv python tools/ncu_step.py --decode > /dev/null 2>&1
ls -la gpurun_out
