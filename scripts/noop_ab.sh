#!/bin/bash
# Fixed-clock (ncu --clock-control base) comparison of the GEMM with its real epilogue and with a no-op
# epilogue (DMPQ_EPI_NOOP): separates epilogue interference from power/clock effects (development).
M="gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second,l1tex__data_bank_reads.avg.pct_of_peak_sustained_elapsed,l1tex__data_bank_writes.avg.pct_of_peak_sustained_elapsed"
for v in ${NOOP_VARIANTS:-"" "-DDMPQ_EPI_NOOP"}; do
    echo "=== variant: $v"
    DMPQ_NVCC_EXTRA="$v" python -c "from paper_2603_18742_b200 import build; build.build(force=True)" || exit 1
    for c in "35552 3072 3072 nvfp4" "35552 12288 3072 nvfp4" "35552 3072 3072 int8"; do
        set -- $c
        ncu --clock-control base --metrics $M -k regex:dmpq_gemm -s 2 -c 1 --csv python scripts/gemm_one.py $1 $2 $3 $4 2>/dev/null | grep -v "^==" | tail -5
    done
done
python -c "from paper_2603_18742_b200 import build; build.build(force=True)"
