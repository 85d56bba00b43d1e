#!/bin/sh
# Install the unmodified reference into baseline/_ref (git-ignored; it travels
# to the GPU box with the snapshot) together with its own test suite, so that
# tests/test_gpu_integration.py can run that suite against the drop-in.
# Needs /root/reference (this container only).
set -e
cd "$(dirname "$0")/.."
if [ ! -d baseline/_ref/wavefuse ]; then
  python -m pip install --no-index --no-build-isolation --no-deps \
    --find-links /opt/wheelhouse --target baseline/_ref /root/reference/pkg
fi
rm -rf baseline/_ref/tests
cp -r /root/reference/pkg/tests baseline/_ref/tests
echo "staged: $(ls baseline/_ref/tests | wc -l) test files in baseline/_ref/tests"
