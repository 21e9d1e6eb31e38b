mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_shard.py tests/test_gpu_parity.py -q -x > gpurun_out/r2_t8.log 2>&1; echo "tests rc=$?"
tail -15 gpurun_out/r2_t8.log
timeout 600 python bench.py --config cfg5 --sharded --steps 3 > gpurun_out/r2_sharded5.json 2>gpurun_out/r2_sharded5.err; echo "sharded rc=$?"
tail -c 1200 gpurun_out/r2_sharded5.json; tail -3 gpurun_out/r2_sharded5.err
