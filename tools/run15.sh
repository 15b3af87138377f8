cd "$GRAFT_REPO_ROOT"
mkdir -p /tmp/ncu
timeout 1500 python bench.py > gpurun_out/bench15.json 2> gpurun_out/bench15.err
echo "bench rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file /tmp/ncu/launches.csv python bench.py --steps 1 --warmup 3 --denoise-steps 5 --no-serving --no-e2e \
  --no-cpu-baseline --profile-range > gpurun_out/ncu_list.log 2>&1
echo "list rc=$?"
python tools/ncu_summary.py list /tmp/ncu/launches.csv > gpurun_out/launch_list_r01.json
gzip -c /tmp/ncu/launches.csv > gpurun_out/launches_r01.csv.gz
SD_NO_GRAPH=1 SD_NVTX=1 timeout 1200 ncu --set full --clock-control none --import-source on --profile-from-start off \
  --nvtx --nvtx-include "conv/" -o /tmp/ncu/conv_full python tools/ncu_step.py > gpurun_out/ncu_conv.log 2>&1
echo "conv rc=$?"
python tools/ncu_summary.py rep /tmp/ncu/conv_full.ncu-rep > gpurun_out/conv_full_summary.jsonl
ncu -i /tmp/ncu/conv_full.ncu-rep --page raw --csv | gzip > gpurun_out/conv_full_raw.csv.gz
ls -la /tmp/ncu gpurun_out
