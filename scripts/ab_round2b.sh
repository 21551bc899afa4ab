#!/bin/bash
# Session A/B (development): Hadamard quantizer stage-1 form and paired 128-B epilogue staging.
set -x
mkdir -p gpurun_out
B() { DMPQ_NVCC_EXTRA="$1" python -c "from paper_2603_18742_b200 import build; build.build(force=True)" || exit 1; }
B "-DDMPQ_EPI_PAIR=1"
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/ab_parity_pair.log 2>&1; echo "parity pair rc=$?" >> gpurun_out/ab_parity_pair.log
for i in 1 2; do
  for v in "-DDMPQ_EPI_PAIR=1" "-DDMPQ_EPI_PAIR=0"; do
    B "$v"; DMPQ_NVCC_EXTRA="$v" timeout 300 python scripts/gemm_variants.py >> gpurun_out/ab_gemm_pair.log 2>&1
  done
  for v in "-DDMPQ_HAD_S1_MIXED=1" "-DDMPQ_HAD_S1_MIXED=0"; do
    B "$v"; echo "=== $v" >> gpurun_out/ab_had_s1.log; timeout 300 python scripts/had_ab.py >> gpurun_out/ab_had_s1.log 2>&1
  done
done
