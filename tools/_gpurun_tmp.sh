mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-serving > gpurun_out/ab.json 2>gpurun_out/ab.err
python -c "
import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);k=d['kernels']
print(round(d['value'],4),round(d['ms_per_step'],1),d['clocks']['sm_mhz'],{a:round(b['ms_per_step'],1) for a,b in k.items()})"
timeout 300 ncu --set full --import-source on --clock-control none -k regex:gemm_kernel -s 3 -c 1 -o gpurun_out/geglu0 python tools/kbench.py --only gemm --pick 0 --reps 2 > gpurun_out/ncu_geglu.log 2>&1
ls -la gpurun_out/
