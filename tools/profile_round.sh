#!/bin/bash
# ncu captures behind profiles/rNN_* (run on the GPU box, one ncu per call;
# each command is first run without ncu and must exit 0).
#   tools/profile_round.sh launches <cfg>      launch list of the bench command
#   tools/profile_round.sh full <cfg> <stage> <kernel-regex> [skip] [count] [tag]
#                                              --set full capture (tools/prof_stage.py)
set -e
mkdir -p gpurun_out
case "$1" in
launches)
    cfg=$2
    python bench.py --config "$cfg" --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-parity --no-by-config > gpurun_out/plain_$cfg.json
    CQG_NO_GRAPH=${NO_GRAPH:-0} ncu --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file gpurun_out/launches_$cfg.csv \
        python bench.py --config "$cfg" --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-parity --no-by-config > gpurun_out/ncu_launch_$cfg.log 2>&1
    ;;
full)
    cfg=$2; stage=$3; kre=$4; skip=${5:-0}; count=${6:-1}; tag=${7:-$stage}
    python tools/prof_stage.py --config "$cfg" --stage "$stage" > gpurun_out/plain_${cfg}_$tag.log
    ncu --set full --import-source on --clock-control none -k "regex:$kre" -s "$skip" -c "$count" \
        -o "gpurun_out/full_${cfg}_${tag}" python tools/prof_stage.py --config "$cfg" --stage "$stage" \
        > gpurun_out/ncu_full_${cfg}_$tag.log 2>&1
    ;;
esac
