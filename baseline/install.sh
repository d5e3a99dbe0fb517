#!/usr/bin/env bash
# Installs the UNMODIFIED reference package (`hybridscale`, /root/reference/pkg) into
# baseline/_ref (git-ignored; it travels to the GPU box with the gpurun snapshot).  The build
# writes into its source tree (Cython extension), so it installs from a scratch copy; the
# offline wheelhouse has no numpy/pyyaml wheels (the image already has both), hence --no-deps.
# The reference's demo config and fixture tables are copied beside the package so that
# configs/demo.yaml resolves its `../tables/*.csv` paths (tests/test_integration_gpu.py).
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
SRC="${REFERENCE_PKG:-/root/reference/pkg}"
DEST="$HERE/_ref"
if [ ! -d "$SRC" ]; then
  echo "reference tree absent: using the prebuilt baseline/_ref if any"; exit 0
fi
if [ -f "$DEST/hybridscale/__init__.py" ] && [ -f "$DEST/configs/demo.yaml" ] && [ "${1:-}" != "--force" ]; then
  exit 0
fi
SCRATCH="$(mktemp -d)"
trap 'rm -rf "$SCRATCH"' EXIT
cp -r "$SRC" "$SCRATCH/pkg"
rm -rf "$DEST"
python3 -m pip install --quiet --no-index --no-build-isolation --no-deps \
  --find-links /opt/wheelhouse --target "$DEST" "$SCRATCH/pkg"
cp -r "$SRC/configs" "$SRC/tables" "$DEST/"
PYTHONPATH="$DEST" python3 -c "import hybridscale; assert hybridscale.KERNEL_BACKEND == 'cython'; print('baseline/_ref: hybridscale', hybridscale.__version__, 'backend', hybridscale.KERNEL_BACKEND)"
