#!/bin/bash
# One GPU session: the GPU tests named by $TESTS (default: all), then the
# commands in $EXTRA. Logs under gpurun_out/.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,memory.total,clocks.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 1500 python -m pytest ${TESTS:-tests} -m gpu -q -rf > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
if [ -n "$EXTRA" ]; then bash -c "$EXTRA" > gpurun_out/extra.log 2>&1; echo "extra rc=$?" >> gpurun_out/extra.log; fi
