#!/bin/bash
# Round-2b evidence pass, part 2: compute-sanitizer (raw tails kept) and the dense full-size race
# guard on the current quantizer and on the round-2-start quantizer (scratch copy, no proxy fence).
mkdir -p gpurun_out/r2b
S=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck synccheck racecheck; do
  timeout 1200 $S --tool $tool python scripts/sanitize_small.py > gpurun_out/r2b/san_$tool.raw 2>&1
  echo "rc=$?" >> gpurun_out/r2b/san_$tool.raw
done
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -m gpu -k dense_all_rows > gpurun_out/r2b/dense_current.log 2>&1
cp paper_2603_18742_b200/csrc/quant_had.cu /tmp/qh_keep.cu
cp scratch/quant_had_round2_start.cu paper_2603_18742_b200/csrc/quant_had.cu
python -c "from paper_2603_18742_b200 import build; build.build(force=True)"
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -m gpu -k dense_all_rows > gpurun_out/r2b/dense_round2_start.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "dense_rows" > gpurun_out/r2b/dense_rows_round2_start.log 2>&1
cp /tmp/qh_keep.cu paper_2603_18742_b200/csrc/quant_had.cu
python -c "from paper_2603_18742_b200 import build; build.build(force=True)"
