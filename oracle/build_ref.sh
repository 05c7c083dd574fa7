#!/usr/bin/env bash
# Install the UNMODIFIED reference package (pure Python + numpy) into
# oracle/_ref so the GPU box, where /root/reference does not exist, can time
# the reference's own nrx_forward as the CPU baseline (bench.py) — the
# Python analogue of compiling a C reference from its sources.  Built from a
# copy under /tmp because setuptools writes into the source tree; outputs go
# only to oracle/_ref (git-ignored, shipped to the GPU box by gpurun).
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
SRC="${NRX_REFERENCE_PKG:-/root/reference/pkg}"
if [ ! -d "$SRC" ]; then
  echo "reference source $SRC not present; keeping existing oracle/_ref" >&2
  exit 0
fi
TMP="$(mktemp -d)"
trap 'rm -rf "$TMP"' EXIT
cp -r "$SRC" "$TMP/pkg"
rm -rf "$HERE/_ref"
python -m pip install --quiet --no-index --no-build-isolation --no-deps --target "$HERE/_ref" "$TMP/pkg"
python -c "import sys; sys.path.insert(0, '$HERE/_ref'); import nrxsim; print('oracle/_ref: nrxsim', nrxsim.__version__)"
