#!/bin/bash
# Install the UNMODIFIED reference package (stereonorm 0.1.0, pure Python) into
# baseline/_ref for bench.py's reference arm.  The build writes egg-info into
# its source tree, so it builds from a copy under /tmp (/root/reference is
# read-only); numpy/scipy/pillow come from the image (--no-deps).
set -eu
cd "$(dirname "$0")/.."
rm -rf /tmp/stereonorm_src baseline/_ref
cp -r /root/reference/pkg /tmp/stereonorm_src
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
  --target baseline/_ref /tmp/stereonorm_src
python -c "import sys; sys.path.insert(0, 'baseline/_ref'); import stereonorm; print('installed', stereonorm.__version__, stereonorm.__file__)"
