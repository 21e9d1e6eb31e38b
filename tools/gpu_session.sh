mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_prune.py tests/test_gpu_parity.py tests/test_gpu_batch.py -q -x > gpurun_out/r2_t7.log 2>&1; echo "tests rc=$?"
tail -5 gpurun_out/r2_t7.log
for i in 1 2; do timeout 300 python bench.py --no-by-config --no-cpu-baseline > gpurun_out/r2_bench_cfg2c.json 2> gpurun_out/r2_bench_cfg2c.err; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/r2_bench_cfg2c.json').read().strip().splitlines()[-1])
print(d['value'], d['e2e']['value'], d['stage_ms_last_step'], {k:round(v['ms_per_step'],4) for k,v in d['kernels'].items()}, d['parity']['ok'])"; done
