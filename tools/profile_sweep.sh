# --set full capture of the isolated dense sweep (cqg_bench_sweep) on cfg3 / cfg5
set -e
mkdir -p gpurun_out
for c in ${CONFIGS:-cfg3 cfg5}; do
  python tools/prof_stage.py --config $c --stage sweep > gpurun_out/plain_${c}_sweep.log
  # the Lloyd loop's WALK sweeps run inside a conditional CUDA graph, which ncu
  # does not profile kernel by kernel: skip only the bench's warm-up launch
  skip=1
  ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
      -k "regex:sweep_kernel<.int.1," -s "$skip" -c 1 -o gpurun_out/full_${c}_sweepdense \
      python tools/prof_stage.py --config $c --stage sweep > gpurun_out/ncu_${c}_sweep.log 2>&1
done
