#!/bin/bash
# Quick GPU pass: parity tests, both bench workloads, stage traces.
#   gpurun --timeout 900 -- 'bash tools/gpu_quick.sh <tag>'
TAG=${1:-quick}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 600 python -m pytest tests -m gpu -x -q --timeout 120 > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python bench.py --cpu-seconds 0 > $OUT/bench.json 2> $OUT/bench.err
timeout 300 python bench.py --workload k16 --cpu-seconds 0 --hyperband-r 0 > $OUT/bench_k16.json 2> $OUT/bench_k16.err
timeout 120 python tools/trace_step.py > $OUT/trace.txt 2>&1
timeout 120 python tools/trace_step.py --workload k16 > $OUT/trace_k16.txt 2>&1

timeout 120 python tools/trace_step.py --warm > $OUT/trace_warm.txt 2>&1
exit 0
