#!/bin/bash
# Round-2 evidence pass: bench lines (default config1, config2, config3, config0,
# reference arms), smoke, warm ncu launch lists of one step, full captures of the
# top kernels.     gpurun --timeout 3000 -- 'bash tools/gpu_evidence_r2.sh <tag>'
TAG=${1:-r2ev}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/smi.txt
for w in config1 config2 config3; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --cache-control none --csv \
    --log-file $OUT/launches_$w.csv python tools/cnn_profile_step.py $w > $OUT/launches_$w.log 2>&1
done
for w in config1 config2 config3; do
  python tools/traffic_summary.py $OUT/launches_$w.csv $w > $OUT/traffic_$w.txt 2>&1
done
cp profiles/ncu_traffic.json $OUT/ncu_traffic.json
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "rc=$?" >> $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench_config1.json 2> $OUT/bench_config1.err
timeout 900 python bench.py --workload config2 > $OUT/bench_config2.json 2> $OUT/bench_config2.err
timeout 900 python bench.py --workload config3 > $OUT/bench_config3.json 2> $OUT/bench_config3.err
timeout 600 python bench.py --workload config0 > $OUT/bench_config0.json 2> $OUT/bench_config0.err
timeout 600 python bench.py --workload config0 --precision f64 --hyperband-r 0 --hyperband-ref-r 0 > $OUT/bench_config0_f64.json 2> $OUT/bench_config0_f64.err
timeout 300 python bench.py --impl reference > $OUT/bench_config1_reference.json 2> $OUT/bench_config1_reference.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_conv_gemm" \
  --launch-skip 20 --launch-count 6 -o $OUT/config2_gemm python tools/cnn_profile_step.py config2 > $OUT/ncu_c2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_bn_bwd|k_dw_wgrad" \
  --launch-skip 40 --launch-count 4 -o $OUT/config1_top python tools/cnn_profile_step.py config1 > $OUT/ncu_c1.log 2>&1
exit 0
