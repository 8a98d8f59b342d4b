#!/bin/bash
# ncu --set full captures of the HBM-bound conv-path kernels of one config1 step.
#   gpurun -- 'bash tools/ncu_cnn_ops.sh <tag> [workload]'
TAG=${1:-ops}
WL=${2:-config1}
OUT=gpurun_out/$TAG
mkdir -p $OUT
cap() {  # name regex skip count
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$2" \
    --launch-skip $3 --launch-count $4 -o $OUT/$1 python tools/cnn_profile_step.py $WL > $OUT/$1.log 2>&1
}
cap bn_bwd_reduce k_bn_bwd_reduce 47 3
cap dw_wgrad k_dw_wgrad 14 3
cap bn_stats k_bn_stats 0 4
cap bn_apply k_bn_apply 0 4
cap opt k_opt 0 1
exit 0
