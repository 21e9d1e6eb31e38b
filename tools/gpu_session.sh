mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_refsuite.py tests/test_gpu_cpp.py tests/test_gpu_exact.py tests/test_gpu_parity.py tests/test_gpu_sampling.py -m gpu -q > gpurun_out/r2_t5.log 2>&1; echo "tests rc=$?"
tail -40 gpurun_out/r2_t5.log
