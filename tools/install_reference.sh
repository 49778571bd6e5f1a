#!/bin/sh
# Installs the UNMODIFIED reference package into baseline/_ref (git-ignored,
# travels to the GPU box with gpurun) plus a copy of its test files, for
# tests/test_reference_suite_gpu.py.  The reference's build writes into its
# source tree, so it is installed from a copy under /tmp.
set -e
cd "$(dirname "$0")/.."
rm -rf /tmp/nao_refpkg baseline/_ref
cp -r /root/reference/pkg /tmp/nao_refpkg
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target baseline/_ref /tmp/nao_refpkg
mkdir -p baseline/_ref/tests
cp -r /root/reference/pkg/tests/* baseline/_ref/tests/
echo "reference installed in baseline/_ref"
