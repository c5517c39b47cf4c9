#!/usr/bin/env bash
# Install the UNMODIFIED reference (spheregrid, pure Python) into baseline/_ref for
# `bench.py --impl reference`.  /root/reference is read-only and setuptools writes build
# files next to the sources, so the install runs from a scratch copy.  Offline: no index,
# the wheelhouse only; numpy/scipy are already in the image, hence --no-deps.
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
SRC="${1:-/root/reference/pkg}"
TMP="$(mktemp -d)"
trap 'rm -rf "$TMP"' EXIT
cp -r "$SRC" "$TMP/pkg"
rm -rf "$ROOT/baseline/_ref"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$ROOT/baseline/_ref" "$TMP/pkg"
python - "$ROOT/baseline/_ref" <<'PY'
import sys
sys.path.insert(0, sys.argv[1])
import spheregrid
assert spheregrid.__file__.startswith(sys.argv[1]), spheregrid.__file__
print("reference installed:", spheregrid.__file__, spheregrid.__version__)
PY
