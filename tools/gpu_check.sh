#!/bin/bash
# One GPU-box pass: build check, GPU parity tests, smoke, bench lines, ncu.
# Usage (from this container): gpurun --timeout 1500 -- 'bash tools/gpu_check.sh [tag]'
set -x
TAG=${1:-run}
OUT=gpurun_out/$TAG
mkdir -p $OUT $OUT/k16
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
timeout 600 python -m pytest tests -m gpu -x -q --timeout 120 > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 400 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 400 python bench.py --workload k16 --cpu-seconds 0 --hyperband-r 0 > $OUT/bench_k16.json 2> $OUT/bench_k16.err
timeout 400 python bench.py --workload wide16 --cpu-seconds 0 --hyperband-r 0 > $OUT/bench_wide16.json 2> $OUT/bench_wide16.err
timeout 300 python bench.py --impl reference --steps 20 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $OUT/launches.csv python tools/profile_step.py --steps 20 > $OUT/ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_ -s 30 -c ${NCU_FULL_COUNT:-4} \
    -o $OUT/full python tools/profile_step.py --steps 20 > $OUT/ncu_full.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
    --log-file $OUT/k16/launches.csv python tools/profile_step.py --workload k16 --steps 20 > $OUT/ncu_launch_k16.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_ -s 30 -c 2 \
    -o $OUT/k16/full python tools/profile_step.py --workload k16 --steps 20 > $OUT/ncu_full_k16.log 2>&1
exit 0
