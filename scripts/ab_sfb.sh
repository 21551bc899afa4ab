#!/bin/bash
# A/B (development): SFB row tiles multicast inside the CTA pair (DMPQ_SFB_MC) vs loaded by both CTAs.
mkdir -p gpurun_out
B() { DMPQ_NVCC_EXTRA="$1" python -c "from paper_2603_18742_b200 import build; build.build(force=True)" || exit 1; }
B ""
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_block_parity.py -x -q -m gpu > gpurun_out/sfb_parity.log 2>&1; echo "rc=$?" >> gpurun_out/sfb_parity.log
for i in 1 2; do
  for v in "-DDMPQ_SFB_MC=1" "-DDMPQ_SFB_MC=0"; do
    B "$v"; DMPQ_NVCC_EXTRA="$v" timeout 300 python scripts/gemm_variants.py >> gpurun_out/sfb_gemm.log 2>&1
  done
done
B ""
