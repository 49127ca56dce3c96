#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_fp8.py -q -s > gpurun_out/fp8_tests.log 2>&1; echo "tests rc=$?"
grep -E "fp8 max|passed|failed|Error" gpurun_out/fp8_tests.log | tail -16
