#!/bin/bash
# A/B (development): 4-CTA clusters with B / SFB TMA multicast (DMPQ_GEMM_CLUSTER=4) vs CTA pairs.
mkdir -p gpurun_out
DMPQ_GEMM_CLUSTER=4 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "gemm" > gpurun_out/cl4_parity.log 2>&1
echo "rc=$?" >> gpurun_out/cl4_parity.log
if grep -q "rc=0" gpurun_out/cl4_parity.log; then
  for i in 1 2; do
    for c in 2 4; do DMPQ_GEMM_CLUSTER=$c timeout 300 python scripts/gemm_variants.py | sed "s/^/cl$c /" >> gpurun_out/cl4_gemm.log 2>&1; done
  done
  for i in 1 2; do
    for c in 2 4; do echo "=== cluster $c" >> gpurun_out/cl4_bench.log; DMPQ_GEMM_CLUSTER=$c timeout 400 python bench.py --no-cpu-baseline >> gpurun_out/cl4_bench.log 2>/dev/null; done
  done
fi
