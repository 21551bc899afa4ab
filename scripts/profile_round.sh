#!/bin/bash
# Profiling pass for profiles/<round>/ (run under gpurun; one GPU, never multi-rank under ncu).
#   bash scripts/profile_round.sh [quant]     (quant: launch list + quantizer captures only)
set -x
OUT=gpurun_out
MODE=$1
# launch list of the bench (every kernel of 2 timed + 3 warm-up steps, eager launches)
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_r1.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-graphs > $OUT/bench_under_ncu.log 2>&1
# one full capture per quantizer configuration of the CogVideoX-5B step
for c in "3072 nvfp4 had" "12288 nvfp4 had" "3072 int8 had" "12288 int8 had" "3072 nvfp4 had ln" "3072 both had ln" \
         "3072 nvfp4 plain" "12288 int8 plain"; do
    set -- $c
    ncu --set full --clock-control none --import-source on -k regex:quant_ -s 2 -c 1 \
        -o $OUT/full_quant_$1_$2_$3${4:+_$4} -f python scripts/quant_one.py $1 $2 $3 $4 > /dev/null 2>&1
done
[ "$MODE" = "quant" ] && exit 0
# TDC kernels (bf16 and NVFP4-compressed cache)
for k in tdc_refresh_kernel tdc_skip_kernel tdc_refresh_nvfp4_kernel tdc_skip_nvfp4_kernel; do
    ncu --set full --clock-control none -k regex:$k -s 2 -c 1 -o $OUT/full_$k -f \
        python scripts/kernel_bench.py --tdc > /dev/null 2>&1
done
