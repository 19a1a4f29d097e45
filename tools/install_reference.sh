#!/bin/bash
# Install the UNMODIFIED reference package (hepack) into baseline/_ref (git-
# ignored; it travels to the GPU box with the gpurun snapshot).  Used only by
# tests/test_dropin.py (the drop-in proof), bench.py's cpu_baseline leg and
# `bench.py --impl reference`; the product never imports it.
# The build writes into its source tree, so it installs from a copy under
# /tmp; --no-deps because matplotlib (only its CLI/report modules need it) is
# not in this image.
set -e
cd "$(dirname "$0")/.."
rm -rf /tmp/hepack_src baseline/_ref
cp -r /root/reference/pkg /tmp/hepack_src
python -m pip install --no-index --no-build-isolation --find-links /opt/wheelhouse \
    --target baseline/_ref --no-deps /tmp/hepack_src
python -c "import sys; sys.path.insert(0, 'baseline/_ref'); import hepack, hepack.ntt; print('hepack', hepack.__file__, 'numba', hepack.ntt._HAVE_NUMBA)"
