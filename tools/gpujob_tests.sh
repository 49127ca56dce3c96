#!/bin/bash
# GPU test job: the whole -m gpu suite with per-test durations (analysis helper)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout ${T:-1500} python -m pytest ${ARGS:-tests} -m gpu -q -x --durations=25 > gpurun_out/gputests.log 2>&1
echo "rc=$?" >> gpurun_out/gputests.log
tail -40 gpurun_out/gputests.log
