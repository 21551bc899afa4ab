#!/bin/bash
# Round-2b profiling pass (paired epilogue staging, quantizer fence + mixed stage 1) (run under gpurun; one GPU, never multi-rank under ncu):
#   launch list of the default bench (graphs off so every launch is visible) + one full capture per
#   top kernel of the CogVideoX-5B step. Summarise here with: python scripts/summarize_ncu.py round2b
OUT=gpurun_out
mkdir -p $OUT
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_r1.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-graphs > $OUT/bench_under_ncu.log 2>&1
for c in "35552 3072 3072 int8" "35552 12288 3072 int8" "35552 3072 12288 int8" "35552 3072 3072 nvfp4" \
         "35552 12288 3072 nvfp4" "35552 3072 12288 nvfp4" "35552 3072 3072 nvfp4 res" "35552 3072 3072 int8 res"; do
    set -- $c
    ncu --set full --clock-control none --import-source on -k regex:dmpq_gemm -s 2 -c 1 \
        -o $OUT/full_${4}_$1_$2_$3${5:+_$5} -f python scripts/gemm_one.py $1 $2 $3 $4 $5 > /dev/null 2>&1
done
for c in "3072 nvfp4 had" "12288 nvfp4 had" "3072 int8 had" "12288 int8 had" "3072 nvfp4 had ln" "3072 both had ln" \
         "3072 int8 had ln"; do
    set -- $c
    ncu --set full --clock-control none --import-source on -k regex:quant_ -s 2 -c 1 \
        -o $OUT/full_quant_$1_$2_$3${4:+_$4} -f python scripts/quant_one.py $1 $2 $3 $4 > /dev/null 2>&1
done
for k in NONE; do [ "$k" = NONE ] && continue
    ncu --set full --clock-control none -k regex:$k -s 2 -c 1 -o $OUT/full_$k -f \
        python scripts/kernel_bench.py --tdc > /dev/null 2>&1
done
ls -la $OUT/*.ncu-rep | wc -l
