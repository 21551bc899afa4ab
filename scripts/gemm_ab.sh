#!/bin/bash
# A/B of gemm.cu compile-time variants (development): GEMM microbenchmarks at the C2/C4 shapes.
#   bash scripts/gemm_ab.sh "-DDMPQ_GEMM_PREFETCH=0" "-DDMPQ_GEMM_PREFETCH=1" ...
for v in "$@"; do
    echo "=== variant: $v"
    DMPQ_NVCC_EXTRA="$v" python -c "from paper_2603_18742_b200 import build; build.build(force=True)" || exit 1
    python scripts/kernel_bench.py --gemm --shapes c2,c4 $GEMM_AB_ARGS
done
python -c "from paper_2603_18742_b200 import build; build.build(force=True)"
