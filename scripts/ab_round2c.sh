#!/bin/bash
# Session A/B (development): partitioned A prefetch (DMPQ_GEMM_PREFETCH=3) on top of paired staging;
# stage-1 diagnostic; parity of the candidate build.
mkdir -p gpurun_out
B() { DMPQ_NVCC_EXTRA="$1" python -c "from paper_2603_18742_b200 import build; build.build(force=True)" || exit 1; }
B "-DDMPQ_HAD_S1_MIXED=1"
timeout 300 python scripts/diag_s1.py > gpurun_out/diag_s1.log 2>&1
for i in 1 2; do
  for v in "-DDMPQ_EPI_PAIR=1 -DDMPQ_HAD_S1_MIXED=0" "-DDMPQ_EPI_PAIR=1 -DDMPQ_HAD_S1_MIXED=0 -DDMPQ_GEMM_PREFETCH=3"; do
    B "$v"; DMPQ_NVCC_EXTRA="$v" timeout 300 python scripts/gemm_variants.py >> gpurun_out/ab_gemm_pf3.log 2>&1
  done
done
B "-DDMPQ_EPI_PAIR=1 -DDMPQ_HAD_S1_MIXED=0 -DDMPQ_GEMM_PREFETCH=3"
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_block_parity.py -x -q -m gpu > gpurun_out/ab_parity_pf3.log 2>&1; echo "rc=$?" >> gpurun_out/ab_parity_pf3.log
