# one GPU session: the -m gpu suite, then the default bench line and cfg5.
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/r2_gputests.log 2>&1; echo "tests rc=$?"
tail -40 gpurun_out/r2_gputests.log
timeout 300 python bench.py --steps 10 --warmup 3 > gpurun_out/r2_bench_cfg2.json 2> gpurun_out/r2_bench_cfg2.err; echo "bench rc=$?"
tail -c 1500 gpurun_out/r2_bench_cfg2.json; tail -5 gpurun_out/r2_bench_cfg2.err
