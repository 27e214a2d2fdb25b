#!/usr/bin/env bash
# Install the UNMODIFIED reference package into baseline/_ref (git-ignored,
# travels to the GPU box with the snapshot): bench.py --impl reference and
# the cpu_baseline of the N=1 line time the reference's own CPU path from
# there.  pip builds the reference's Cython kernel extension (_core) from a
# scratch copy of /root/reference/pkg (the source tree is read-only); nothing
# of the reference is copied into tracked files.
set -euo pipefail
REF=${1:-/root/reference/pkg}
ROOT=$(cd "$(dirname "$0")/.." && pwd)
if [ ! -d "$REF" ]; then
    echo "build_ref: no reference at $REF (GPU box): using the prebuilt baseline/_ref"
    exit 0
fi
TMP=$(mktemp -d)
trap 'rm -rf "$TMP"' EXIT
cp -r "$REF" "$TMP/pkg"
rm -rf "$ROOT/baseline/_ref"
python -m pip install --quiet --no-index --no-build-isolation --find-links /opt/wheelhouse \
    --no-deps --target "$ROOT/baseline/_ref" "$TMP/pkg"
MICROMACRO_BACKEND=compiled PYTHONPATH="$ROOT/baseline/_ref" python -c \
    "import micromacro._kernels as K; assert K.backend_name == 'compiled', K.backend_name; print('build_ref: reference installed, backend', K.backend_name)"
