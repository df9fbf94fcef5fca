#!/bin/bash
# Vendor the unmodified reference (roboserve) as TEST INFRASTRUCTURE under
# baseline/_ref/ (git-ignored; travels to the GPU box with gpurun): the
# installed package, its test suite and scratch_fig4.py.  Used only by
# tests/test_gpu_reference_vendored.py and tools/call_latency.py (the
# reference timed beside the drop-in); never by the product.
set -e
cd "$(dirname "$0")/.."
REF=${1:-/root/reference}
[ -d "$REF/pkg" ] || { echo "no reference at $REF"; exit 1; }
rm -rf /tmp/kr_refsrc baseline/_ref
cp -r "$REF/pkg" /tmp/kr_refsrc
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target baseline/_ref /tmp/kr_refsrc -q
mkdir -p baseline/_ref/pkg
cp -r "$REF/pkg/tests" baseline/_ref/pkg/tests
cp "$REF/pkg/scratch_fig4.py" baseline/_ref/pkg/scratch_fig4.py
echo "vendored roboserve into baseline/_ref"
