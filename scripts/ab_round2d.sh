#!/bin/bash
# Session A/B (development): the quantizer's proxy fence before the buffer release (race fix),
# the FHADD stage 1, and paired epilogue staging, measured in the full CogVideoX-5B step
# (bench breakdown, same box, interleaved) and in isolation (had_ab).
mkdir -p gpurun_out
B() { DMPQ_NVCC_EXTRA="$1" python -c "from paper_2603_18742_b200 import build; build.build(force=True)" || exit 1; }
for v in "-DDMPQ_HAD_S1_MIXED=1" ""; do
  B "$v"; echo "=== parity [$v]" >> gpurun_out/ab2d_parity.log
  timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "hadamard or adversarial" >> gpurun_out/ab2d_parity.log 2>&1
done
for v in "" "-DDMPQ_HAD_NO_PROXY_FENCE"; do
  B "$v"; echo "=== had_ab [$v]" >> gpurun_out/ab2d_had.log; timeout 300 python scripts/had_ab.py >> gpurun_out/ab2d_had.log 2>&1
done
for i in 1 2; do
  for v in "" "-DDMPQ_HAD_S1_MIXED=1" "-DDMPQ_HAD_NO_PROXY_FENCE" "-DDMPQ_EPI_PAIR=0"; do
    B "$v"; echo "=== bench [$v]" >> gpurun_out/ab2d_bench.log
    timeout 400 python bench.py --no-cpu-baseline >> gpurun_out/ab2d_bench.log 2>/dev/null
  done
done
B ""
