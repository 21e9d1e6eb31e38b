# one GPU session: the -m gpu suite, then the default bench line
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --durations=8 > gpurun_out/r2_gputests.log 2>&1; echo "tests rc=$?"
tail -25 gpurun_out/r2_gputests.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2_bench_cfg2b.json 2> gpurun_out/r2_bench_cfg2b.err; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/r2_bench_cfg2b.json').read().strip().splitlines()[-1])
print(d['value'], d['stage_ms_last_step'], {k:v['ms_per_step'] for k,v in d['kernels'].items()}, d['parity']['ok'])"
